set -x
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -2
timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 256,512,768 2>&1 | grep -v "epilogue\|prologue" | tail -36
