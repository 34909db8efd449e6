FRB_LIB=$PWD/paper_2305_07030_b200/lib/libfrb200_ug.so timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -2
for v in "" _ug; do
  L=$PWD/paper_2305_07030_b200/lib/libfrb200$v.so
  echo "== $v"; FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768,512 2>&1 | grep -v "epilogue\|prologue"
done
