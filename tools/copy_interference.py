"""Does PCIe traffic on the copy engines slow the solve?  C3 solve times (CUDA events) alone and with
concurrent H2D + D2H copies of the e2e loop's size (Ω-compact f and u, 205 MB each way) in flight."""
import os, sys, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import workloads as W
from paper_2404_15249_b200 import KFBI
prob = W.C3()
k = KFBI(prob)
pz, pq = k.points("ctrl"), k.points("isect")
x = prob.lo + np.arange(prob.n + 1) * prob.h
X, Y = np.meshgrid(x, x, indexing="ij")
f = lambda *a: W.f_exact(prob.kappa, *a)
dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
g, fg, fq, fz = dev(W.u_exact(*pz.T)), dev(f(X, Y).ravel()), dev(f(*pq.T)), dev(f(*pz.T))
u = torch.empty(k.n_nodes, dtype=torch.float64, device="cuda")
nb = 205_000_000 // 8
hA = torch.empty(nb, dtype=torch.float64).pin_memory(); dA = torch.empty(nb, dtype=torch.float64, device="cuda")
hB = torch.empty(nb, dtype=torch.float64).pin_memory(); dB = torch.empty(nb, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timed(copies, reps=5):
    ts = []
    for _ in range(reps):
        if copies:
            with torch.cuda.stream(s1): dA.copy_(hA, non_blocking=True)
            with torch.cuda.stream(s2): hB.copy_(dB, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); k.solve(g, fg, fq, fz, u=u); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
        torch.cuda.synchronize()
    return ts
timed(False, 2)
print("alone      ", ["%.2f" % t for t in timed(False)])
print("with copies", ["%.2f" % t for t in timed(True)])
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s1); dA.copy_(hA, non_blocking=True); e1.record(s1); e1.synchronize(); print("H2D 205 MB ms", e0.elapsed_time(e1))
e0.record(s2); hB.copy_(dB, non_blocking=True); e1.record(s2); e1.synchronize(); print("D2H 205 MB ms", e0.elapsed_time(e1))
