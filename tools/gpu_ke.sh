# kElem (F1 elements in flight) variants on c2 (256 threads) and one C3 wave
for v in "" _ke2 _ke4 _ke5 _ke6; do
  L=$PWD/paper_2305_07030_b200/lib/libfrb200$v.so
  echo "== $v"
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 15 --P 222 --teams 256 2>&1 | grep "T=\|F1"
  FRB_LIB=$L timeout 300 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | grep "T=\|F1"
done
