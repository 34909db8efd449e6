# after the bulk-copy halo exchange: parity + phase profiles
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | tail -14
timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | tail -14
