"""Summarise an ncu SASS source page CSV: opcode mix, stall reasons, hot spots."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr)]
def num(x):
    try: return float(x.replace(',', ''))
    except Exception: return 0.0
tot_exec = sum(num(d['Instructions Executed']) for d in data)
tot_samp = sum(num(d['Warp Stall Sampling (All Samples)']) for d in data)
print(f"instructions executed (warp) {tot_exec:.4g}, stall samples {tot_samp:.4g}")
op = collections.Counter(); ops = collections.Counter()
for d in data:
    o = d['Source'].split()[0] if d['Source'] else '?'
    if o.startswith('@'): o = d['Source'].split()[1]
    base = o.split('.')[0]
    op[base] += num(d['Instructions Executed']); ops[base] += num(d['Warp Stall Sampling (All Samples)'])
print("opcode          exec%   stall%")
for o, v in op.most_common(25):
    print(f"{o:14s} {100*v/tot_exec:6.2f} {100*ops[o]/max(tot_samp,1):7.2f}")
stalls = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
sc = {s: sum(num(d[s]) for d in data) for s in stalls}
print("stall reasons:", {k: round(100*v/max(tot_samp,1),1) for k, v in sorted(sc.items(), key=lambda kv: -kv[1])[:10]})
# hot windows of 40 instructions
win = 60
best = []
for i in range(0, len(data), win):
    chunk = data[i:i+win]
    best.append((sum(num(d['Warp Stall Sampling (All Samples)']) for d in chunk), sum(num(d['Instructions Executed']) for d in chunk), i))
best.sort(reverse=True)
for s, e, i in best[:8]:
    print(f"window @{i:5d} ({data[i]['Address']}): stall {100*s/tot_samp:5.1f}%  exec {100*e/tot_exec:5.1f}%")
