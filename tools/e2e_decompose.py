"""Where does the C3 e2e step go?  Back-to-back Ω-compact (opts.omega_io) solves timed over 30 steps on
the device: (a) no copies, (b) the H2D upload of each step's inputs only, (c) the D2H download only,
(d) both — the pipelined loop of bench.py without its fill and drain."""
import os, sys
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
mask = k.node_mask().reshape(-1).astype(bool)
dev = lambda a: torch.tensor(np.ascontiguousarray(a), device="cuda")
g, fq, fz = dev(W.u_exact(*pz.T)), dev(f(*pq.T)), dev(f(*pz.T))
fc = dev(f(X, Y).ravel()[mask])
u = [torch.empty(k.omega_count(), dtype=torch.float64, device="cuda") for _ in range(2)]
h_in = torch.empty(fc.numel(), dtype=torch.float64).pin_memory()
h_out = [torch.empty(fc.numel(), dtype=torch.float64).pin_memory() for _ in range(2)]
d_in = [torch.empty_like(fc) for _ in range(2)]
s_up, s_dn = torch.cuda.Stream(), torch.cuda.Stream()
st = torch.cuda.current_stream()


def run(up, down, n=30, chunks=1):
    ev_done = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for j in range(n):
        b = j % 2
        if up:
            with torch.cuda.stream(s_up):
                s_up.wait_event(ev_done[1 - b])
                d_in[1 - b].copy_(h_in, non_blocking=True)
        k.solve(g, fc, fq, fz, u=u[b], async_final=True, omega_io=True)
        ev_done[b].record(st)
        if down:
            with torch.cuda.stream(s_dn):
                s_dn.wait_event(ev_done[b])
                for part_h, part_d in zip(h_out[b].chunk(chunks), u[b].chunk(chunks)):
                    part_h.copy_(part_d, non_blocking=True)
    st.wait_stream(s_up)
    st.wait_stream(s_dn)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / n


run(False, False, 3)
for name, up, down, ch in [("no copies", False, False, 1), ("upload only", True, False, 1),
                           ("download only", False, True, 1), ("download 16 chunks", False, True, 16),
                           ("both", True, True, 1), ("no copies again", False, False, 1)]:
    print(f"{name:20s} {run(up, down, chunks=ch):.3f} ms/step")
