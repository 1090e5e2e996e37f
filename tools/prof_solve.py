"""Drive a few full solves of a config for ncu / timing (no output checks):
python tools/prof_solve.py [C3] [reps]  — prints ms per solve (CUDA events)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_15249_b200 import KFBI  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
prob = W.CONFIGS[cfg]()
k = KFBI(prob)
pz, pq = k.points("ctrl"), k.points("isect")
x = prob.lo + np.arange(prob.n + 1) * prob.h
dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
if prob.dim == 2:
    X, Y = np.meshgrid(x, x, indexing="ij")
    fg = dev(W.f_exact(prob.kappa, X, Y).ravel())
    g, fq, fz = dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, *pq.T)), dev(W.f_exact(prob.kappa, *pz.T))
else:
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    fg = dev(W.f_exact(prob.kappa, X, Y, Z).ravel())
    g, fq, fz = dev(W.u_exact(*pz.T)), dev(W.f_exact(prob.kappa, *pq.T)), dev(W.f_exact(prob.kappa, *pz.T))
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for r in range(reps):
    e0.record()
    u, phi, st = k.solve(g, fg, fq, fz)
    e1.record()
    torch.cuda.synchronize()
    print(f"solve {r}: {e0.elapsed_time(e1):.3f} ms, {st}")
