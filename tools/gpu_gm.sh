set -x
timeout 600 python -m pytest tests/test_gpu_parity_full.py -x -q 2>&1 | tail -4
timeout 300 python tools/sanitize_cluster.py 32 200 --check 2>&1 | tail -2
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_gm.json 2>gpurun_out/bench_c3_gm.err; tail -3 gpurun_out/bench_c3_gm.err; python -c "import json; d=json.load(open('gpurun_out/bench_c3_gm.json')); print('c3', d['value'], d['roofline']['frac'], d['e2e']['value'], d['parity_spot_check']['all_bit_equal'])"
