FRB_VIRTUAL_ONLY=1 timeout 600 python tools/phase_profile.py --n 32 --P 9 --teams 768 2>&1 | grep -v "epilogue\|prologue"
timeout 600 python tools/phase_profile.py --n 32 --P 7 --teams 768 2>&1 | head -1
FRB_VIRTUAL_ONLY=1 timeout 1200 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('virtual-only c3', d['value'], d['roofline']['frac'])"
