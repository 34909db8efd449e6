# round 2: parity after the double-buffered exchange, cluster occupancy, C3 phase profile
set -x
./tools/ubench/clusters
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -6
timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | tail -14
timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | tail -14
