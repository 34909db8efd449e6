for c in c3 c4 c5; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_$c.json
  python -c "import json; d=json.load(open('gpurun_out/bench_$c.json')); print('$c', round(d['value'],1), round(d['ms_per_step'],1), round(d['roofline']['frac'],3), round(d['iters_mean']), round(d['e2e']['value'],1), d['config'].get('networks_per_gpu'))"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 2>/dev/null | tail -1 > gpurun_out/bench_ref.json; tail -c 600 gpurun_out/bench_ref.json
