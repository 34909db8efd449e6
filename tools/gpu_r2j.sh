set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 512 2>&1 | grep -v "epilogue\|prologue" | tail -12
FRB_LIB=$PWD/paper_2305_07030_b200/lib/libfrb200_f1pipe.so timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 512 2>&1 | grep -v "epilogue\|prologue" | tail -12
timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | grep -v "epilogue\|prologue" | tail -12
FRB_LIB=$PWD/paper_2305_07030_b200/lib/libfrb200_f1pipe.so timeout 300 python tools/phase_profile.py --n 15 --P 256 --teams 256 2>&1 | head -1
S=/usr/local/cuda/bin/compute-sanitizer
for n in 32 24; do
  timeout 1200 $S --tool racecheck --print-limit 50 python tools/sanitize_cluster.py $n 200 > gpurun_out/sanitize_racecheck_$n.log 2>&1
  echo "n=$n racecheck rc=$?: $(grep -E 'RACECHECK SUMMARY|ERROR SUMMARY|iters' gpurun_out/sanitize_racecheck_$n.log | tr '\n' ' ')"
done
