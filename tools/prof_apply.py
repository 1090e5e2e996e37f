"""Drive a few K_D applies of a config for ncu / timing (no output checks)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads as W
from paper_2404_15249_b200 import KFBI
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
k = KFBI(W.CONFIGS[cfg]())
phi = torch.tensor(W.random_density(k.M, 0), device="cuda")
for _ in range(reps):
    out = k.apply(phi)
torch.cuda.synchronize()
print(k.profile_apply(phi, reps=5))
