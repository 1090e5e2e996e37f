"""Dense sweep in place (test fast solve) vs out of place (solve's Y apply) at C3, for an ncu launch list."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_15249_b200 import KFBI  # noqa: E402

k = KFBI(W.C3())
rhs = torch.randn(k.n_nodes, dtype=torch.float64, device="cuda")
for _ in range(2):
    k.test_fast_solve(rhs)
torch.cuda.synchronize()
