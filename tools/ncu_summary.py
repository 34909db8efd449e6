"""Summarise an ncu report: key raw metrics, stall reasons, hottest CUDA source lines."""
import csv, subprocess, sys, io, collections

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "launch__cluster_dim_x",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__t_sector_hit_rate.pct",
        "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_barrier.ratio"]
for w in want:
    if w in hdr:
        i = hdr.index(w)
        print(f"{w:60s} {vals[i]} {units[i]}")
st = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")]
tot = sum(float(v.replace(",", "")) for _, v in st if v)
top = sorted(((float(v.replace(",", "")) / tot, h.replace("smsp__pcsamp_warps_issue_stalled_", "")) for h, v in st if v), reverse=True)[:10]
print("stalls:", ", ".join(f"{n} {100 * f:.1f}%" for f, n in top))

rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
cur = None
out = []
ts = te = 0.0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if len(r) < 9 or r[0] == "Line No":
        continue
    if r[0] != "" and r[2] == "-":
        try:
            s, e = float(r[4]), float(r[7])
        except ValueError:
            continue
        out.append((s, e, cur, r[0], r[1][:100]))
        ts += s
        te += e
out.sort(reverse=True)
print(f"total stall samples {ts:.0f}, warp instructions {te:.4g}")
for s, e, f, l, src in out[:ntop]:
    print(f"{100 * s / ts:5.1f}% stall {100 * e / te:5.1f}% exec  {f}:{l}  {src.strip()}")
