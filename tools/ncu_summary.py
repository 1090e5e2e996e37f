"""Summarise an ncu --set full report: key metrics + stall reasons per kernel (run here, no GPU)."""
import csv, io, subprocess, sys

rep = sys.argv[1]
KEYS = ['Duration', 'DRAM Throughput', 'Memory Throughput', 'Compute (SM) Throughput', 'Achieved Occupancy',
        'Theoretical Occupancy', 'Registers Per Thread', 'L2 Hit Rate', 'L1/TEX Hit Rate', 'Executed Ipc Active',
        'Warp Cycles Per Issued Instruction', 'L1/TEX Cache Throughput', 'Executed Instructions',
        'Dynamic Shared Memory Per Block', 'Grid Size', 'Block Size']


def run(args):
    return subprocess.run(["ncu", "-i", rep] + args, capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run(["--page", "details", "--csv"]))))
h = det[0]
ki, ii, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
seen = {}
for r in det[1:]:
    if r[mi] in KEYS:
        seen.setdefault((r[ii], r[ki][:60]), {})[r[mi]] = f"{r[vi]} {r[ui]}"
for (i, k), m in seen.items():
    print(f"== [{i}] {k}")
    for key in KEYS:
        if key in m:
            print(f"   {key:38s} {m[key]}")
raw = list(csv.reader(io.StringIO(run(["--page", "raw", "--csv"]))))
h = raw[0]
names = [c for c in h if c.startswith("smsp__pcsamp_warps_issue_stalled_") and not c.endswith("not_issued")]
dram = [c for c in h if c in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
for r in raw[2:]:
    vals = []
    for n in names:
        try:
            vals.append((float(r[h.index(n)].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
    tot = sum(v for v, _ in vals) or 1
    top = ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in sorted(vals, reverse=True)[:6])
    d = ", ".join(f"{c.split('__')[1]}={r[h.index(c)]} {raw[1][h.index(c)]}" for c in dram)
    print(f"-- [{r[h.index('ID')]}] {r[h.index('Kernel Name')][:50]}: stalls: {top}\n      {d}")
