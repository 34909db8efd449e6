# one ncu --set full capture of the relax kernel on the c2 bench (+ launch list)
CFG=${CFG:-c2}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$CFG.csv python bench.py --config $CFG --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; grep -c frb_ gpurun_out/launches_$CFG.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_$CFG python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full_$CFG.log 2>&1; tail -2 gpurun_out/ncu_full_$CFG.log
