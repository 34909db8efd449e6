python -m pytest tests -m gpu -x -q -k "not energy" 2>&1 | tail -2
for T in ${TEAMS:-1024}; do
  python bench.py --no-cpu-baseline --steps 5 --warmup 3 --team-size $T > gpurun_out/bench_T$T.json 2> gpurun_out/bench_T$T.err
  python -c "import json; d=json.load(open('gpurun_out/bench_T$T.json')); print('T=$T c2 nets/s', round(d['value'],1), 'kernel ms', round(d['roofline']['kernel_ms'],2), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],1), d['kernel_ms_per_step'])" || tail -3 gpurun_out/bench_T$T.err
done
python bench.py --config c1 --no-cpu-baseline --steps 5 --warmup 3 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c1 ms', d['ms_per_step'], 'threads', d['config']['cta_threads'])"
if [ "${NCU:-1}" = "1" ]; then
timeout 600 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/prof_quick python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_quick.log 2>&1; tail -1 gpurun_out/ncu_quick.log
fi
