"""Gray–Scott timing (NEXT-2) on the paper's Table configs: grid 128²..1024² with 8..64
Strang steps to T = 1 (reading: Δt = 1/steps; the paper does not state T for the table), GMRES tol 1e-8.
Prints one JSON line per config with the device time of the whole run (setup excluded) and the
paper's RTX 3090 GPU time as context (other hardware)."""
import json
import sys

import torch

import workloads as W
from paper_2404_15249_b200 import GrayScott

PAPER_GPU_S = {128: 0.40, 256: 1.04, 512: 3.29, 1024: 12.07}
cfgs = [(128, 8), (256, 16), (512, 32), (1024, 64)]
if len(sys.argv) > 1:
    cfgs = [c for c in cfgs if c[0] in {int(a) for a in sys.argv[1:]}]
for n, steps in cfgs:
    g = GrayScott(n, 1.0 / steps, W.GS_PARAMS, W.gray_scott_problem, W.gray_scott_initial, tol=1e-8)
    g.step()                      # warm-up (first GMRES cold start); restart from the initial data
    g = GrayScott(n, 1.0 / steps, W.GS_PARAMS, W.gray_scott_problem, W.gray_scott_initial, tol=1e-8)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        g.step()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    u, v = g.fields()
    m = torch.tensor(g.ku.node_mask().astype(bool), device=u.device)
    print(json.dumps({"workload": "gray-scott", "grid": n, "steps": steps, "dt": 1.0 / steps, "run_s": t,
                      "s_per_step": t / steps, "gmres_iters_per_solve": sum(a + b for a, b in g.iters) / (2 * steps),
                      "u_range": [float(u[m].min()), float(u[m].max())], "v_range": [float(v[m].min()), float(v[m].max())],
                      "paper_gpu_s_rtx3090": PAPER_GPU_S[n]}), flush=True)
