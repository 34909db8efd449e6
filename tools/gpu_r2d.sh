# C3 CTA-size experiment: phase profiles at 256 / 512 / 768 threads + parity at each
set -x
timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 256,512,768 2>&1 | tail -42
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -3
