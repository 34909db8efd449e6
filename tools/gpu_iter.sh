# quick iteration: parity tests (energy ledger excluded until implemented), c2 sweep, phase profile
timeout 600 python -m pytest tests -m gpu -x -q -k "not energy" 2>&1 | tail -4
TEAMS=${TEAMS:-512,768,1024} DPR=${DPR:-3400} timeout 600 python tools/sweep_c2.py 2>&1 | tail -8
timeout 300 python tools/phase_profile.py --teams ${PT:-1024} 2>&1 | tail -10
