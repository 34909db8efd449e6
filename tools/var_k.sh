# c2 kernel time of the default library and any libfrb200_<v>.so variants, then a phase profile
for f in paper_2305_07030_b200/lib/libfrb200*.so; do
  export FRB_LIB=$PWD/$f
  echo "== $f"
  TEAMS=256 DPR=8000 timeout 300 python tools/sweep_c2.py 2>&1 | tail -1
done
unset FRB_LIB
timeout 300 python tools/phase_profile.py --teams 256 2>&1 | tail -14
