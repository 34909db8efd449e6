# A/B of variant libraries ($VARIANTS, e.g. "_xg") against the default: one C3 wave (768 threads) and a c2 wave
for v in "" $VARIANTS; do
  L=$PWD/paper_2305_07030_b200/lib/libfrb200$v.so
  echo "== $v"
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | grep "T=\|F1\|A per\|U upd"
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 15 --P 74 --teams 256 2>&1 | grep "T="
done
