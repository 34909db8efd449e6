# full-length parity + C3 phase-profile experiments (CTA size, shadow work)
set -x
timeout 1200 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -6
timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 512,768 2>&1 | tail -28
FRB_LIB=$PWD/paper_2305_07030_b200/lib/libfrb200_noshadow.so timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | tail -14
FRB_LIB=$PWD/paper_2305_07030_b200/lib/libfrb200_noshadow.so timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | tail -14
