"""Top SASS lines by warp-stall samples of an ncu report: python tools/hot.py rep [n]."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out))
h = r[1]
rows = r[2:]
S = h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(x[S]) for x in rows if x[S]) or 1.0
for x in sorted(rows, key=lambda x: -float(x[S] or 0))[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"{float(x[S]) / tot * 100:5.1f}%  {x[0][-5:]} {x[1][:80]}")
