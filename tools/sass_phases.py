"""Split an ncu SASS CSV at BAR instructions and report per-segment cost."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def num(x):
    try: return float(x.replace(',', ''))
    except Exception: return 0.0
tot_s = sum(num(d['Warp Stall Sampling (All Samples)']) for d in data)
tot_e = sum(num(d['Instructions Executed']) for d in data)
seg_s = seg_e = 0.0; start = 0; segs = []
ops = {}
for i, d in enumerate(data):
    seg_s += num(d['Warp Stall Sampling (All Samples)']); seg_e += num(d['Instructions Executed'])
    src = d['Source'].strip()
    o = src.split()[0] if src else ''
    if o.startswith('@'): o = src.split()[1]
    if o.startswith(('DADD','DMUL','DFMA','MUFU','DSETP')):
        ops['fp64'] = ops.get('fp64', 0) + num(d['Instructions Executed'])
    if 'BAR' in o or 'EXIT' in o or i == len(data) - 1:
        segs.append((start, i, seg_s, seg_e, src[:40]))
        seg_s = seg_e = 0.0; start = i + 1
for a, b, s, e, src in segs:
    if s / tot_s > 0.005 or e / tot_e > 0.005:
        print(f"[{a:5d}-{b:5d}] {data[a]['Address']}  stall {100*s/tot_s:5.1f}%  exec {100*e/tot_e:5.1f}%  ends: {src}")
print('fp64 share of executed', ops.get('fp64', 0) / tot_e)
