"""Warp-stall samples aggregated per CUDA source line: python tools/hotsrc.py rep [n]."""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out))
hi = next(i for i, x in enumerate(r) if "Warp Stall Sampling (All Samples)" in x)
h = r[hi]
S = h.index("Warp Stall Sampling (All Samples)")
agg = []
for x in r[hi + 1:]:
    if len(x) > S and x[0]:
        try:
            agg.append((float(x[S] or 0), x[0], x[1]))
        except ValueError:
            continue
tot = sum(a for a, _, _ in agg) or 1.0
for a, ln, src in sorted(agg, reverse=True)[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{a / tot * 100:5.1f}%  L{ln:>5} {src.strip()[:100]}")
