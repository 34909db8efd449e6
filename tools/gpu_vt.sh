for v in "" _vt; do
  L=$PWD/paper_2305_07030_b200/lib/libfrb200$v.so
  echo "== $v"; FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | head -1
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | head -1
done
