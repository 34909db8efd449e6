# C3 baseline: bench line, launch list and one ncu --set full capture of the C3 kernel (one wave of 7 networks)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
nproc
timeout 900 python bench.py --config c3 --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 3000 gpurun_out/bench_c3.json; tail -3 gpurun_out/bench_c3.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_c3 python bench.py --config c3 --limit 7 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_c3.log 2>&1; tail -3 gpurun_out/ncu_full_c3.log
