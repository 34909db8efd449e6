# quick GPU iteration: parity tests, C2 bench, one ncu capture of the top kernel
python -m pytest tests -m gpu -x -q 2>&1 | tail -4
python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('c2 nets/s', round(d['value'],1), 'kernel ms', round(d['roofline']['kernel_ms'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['clocks'], d['kernel_ms_per_step'])" || tail -5 gpurun_out/bench_quick.err
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_quick python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_quick.log 2>&1; tail -1 gpurun_out/ncu_quick.log
fi
