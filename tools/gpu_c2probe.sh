# c2 probes: wave/tail split and CTA size on the current kernel
timeout 600 python tools/tail_probe.py 2>&1 | grep -v Warn
TEAMS=256,384,512 DPR=3400 timeout 600 python tools/sweep_c2.py 2>&1 | grep -v Warn
