"""Per-source-line hot spots of one kernel in an ncu report (all source files):
python tools/hotsrc2.py rep kernel-regex [n].  Columns: % of stall samples, % of executed warp
instructions, file:line, source."""
import csv
import subprocess
import sys

rep, kr = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", "regex:" + kr],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
f, h, agg = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] in ("File Path", "File Name"):
        f = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = r
        S = h.index("Warp Stall Sampling (All Samples)")
        I = h.index("Instructions Executed")
        continue
    if h is None or len(r) <= max(S, I) or not r[0]:
        continue
    try:
        agg.append((float(r[S] or 0), float(r[I] or 0), f"{f}:{r[0]}", r[1]))
    except ValueError:
        pass
ts = sum(a[0] for a in agg) or 1.0
ti = sum(a[1] for a in agg) or 1.0
for s, i, loc, src in sorted(agg, reverse=True)[:n]:
    print(f"{100 * s / ts:5.1f}% {100 * i / ti:5.1f}%  {loc:18s} {src.strip()[:110]}")
