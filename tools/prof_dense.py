"""Time the dense DST path (kfbi_test_fast_solve) for a config."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, workloads as W
from paper_2404_15249_b200 import KFBI
cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
k = KFBI(W.CONFIGS[cfg]())
rhs = torch.rand(k.n_nodes, dtype=torch.float64, device="cuda")
for _ in range(3): k.test_fast_solve(rhs)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(5): k.test_fast_solve(rhs)
e1.record(); e1.synchronize()
print("fast solve ms", e0.elapsed_time(e1) / 5)
