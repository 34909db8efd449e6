# final round-2 measurements: tests, smoke, default bench line (C3, CPU baseline included), c2/c5 lines,
# launch list and ncu --set full of the C3 and c2 kernels
set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 2400 python bench.py --steps 5 --warmup 3 > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err
python -c "import json; d=json.load(open('gpurun_out/final_c3.json')); print('c3', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['parity_spot_check']['all_bit_equal'], d['clocks'])"
timeout 900 python bench.py --config c2 --steps 5 --warmup 3 > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err
python -c "import json; d=json.load(open('gpurun_out/final_c2.json')); print('c2', d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'])"
timeout 1500 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err
python -c "import json; d=json.load(open('gpurun_out/final_c5.json')); print('c5', d['value'], d['roofline']['frac'], d['e2e']['value'])"
#timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/final_prof_c3 python bench.py --config c3 --limit 7 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
#timeout 900 ncu --set full --clock-control none --import-source on -k regex:frb_relax -s 3 -c 1 -f -o gpurun_out/final_prof_c2 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
#ls gpurun_out/final_prof_*
