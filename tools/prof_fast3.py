"""Run the 3D fast solver (dense rows path) a few times on cfg (for ncu launch lists)."""
import sys

import numpy as np
import torch

import workloads as W
from paper_2404_15249_b200 import KFBI

prob = getattr(W, sys.argv[1] if len(sys.argv) > 1 else "C5")()
k = KFBI(prob)
n = prob.n
rhs = np.random.default_rng(0).uniform(-1, 1, (n + 1,) * 3)
for _ in range(int(sys.argv[2]) if len(sys.argv) > 2 else 2):
    v = k.test_fast_solve(rhs)
torch.cuda.synchronize()
print("ok", float(v.abs().max()))
