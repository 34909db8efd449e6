# ncu --set full captures of the relaxation kernel: C3 (one wave of 7 networks) and c2; launch lists
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_c3 python bench.py --config c3 --limit 7 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c3.log 2>&1; tail -2 gpurun_out/ncu_full_c3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_c2.log 2>&1; tail -2 gpurun_out/ncu_full_c2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1; grep -c frb_ gpurun_out/launches_c3.csv
