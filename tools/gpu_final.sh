# final round-2 measurements: tests, smoke, default bench line (C3, CPU baseline included), c2/c4/c5 lines
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python bench.py --steps 5 --warmup 3 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
python -c "import json; d=json.load(open('gpurun_out/final_c3.json')); print('c3', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity_spot_check']['all_bit_equal'], d['gpu_launches'], d['clocks'])"
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
python -c "import json; d=json.load(open('gpurun_out/final_c2.json')); print('c2', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
timeout 1200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err
python -c "import json; d=json.load(open('gpurun_out/final_c4.json')); print('c4', d['value'], d['roofline']['frac'], d['e2e']['value'], d['gpu_launches'])"
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
python -c "import json; d=json.load(open('gpurun_out/final_c5.json')); print('c5', d['value'], d['roofline']['frac'], d['e2e']['value'])"
