# A/B of a variant library against the default: C3 wave (768 and 512 threads) and c2
V=${V:-fs}
for v in "" _$V; do
  L=$PWD/paper_2305_07030_b200/lib/libfrb200$v.so
  echo "== $v"; FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768,512 2>&1 | grep "T="
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | head -1
done
