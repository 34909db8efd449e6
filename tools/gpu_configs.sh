# every BASELINE config on one B200 + the reference arm for c3 and c2
for c in c1 c2 c4 c5; do
  timeout 1500 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/r02_bench_$c.json 2>gpurun_out/r02_bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/r02_bench_$c.json')); print('$c', round(d['value'],1), round(d['ms_per_step'],1), round(d['roofline']['frac'],3), round(d['iters_mean']), round(d['e2e']['value'],1), d['config']['networks_per_gpu'], d['parity_spot_check'])"
done
timeout 2400 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_c3.json 2>gpurun_out/r02_bench_c3.err
python -c "import json; d=json.load(open('gpurun_out/r02_bench_c3.json')); print('c3', round(d['value'],1), round(d['roofline']['frac'],3), round(d['e2e']['value'],1), d['cpu_baseline']['value'], d['clocks'])"
timeout 2400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_c3.json 2>&1; tail -c 600 gpurun_out/r02_bench_reference_c3.json
timeout 900 python bench.py --impl reference --config c2 --steps 3 --warmup 3 > gpurun_out/r02_bench_reference_c2.json 2>&1; tail -c 400 gpurun_out/r02_bench_reference_c2.json
