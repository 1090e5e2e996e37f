"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck, one tool per run):
C1 solve (every 2D kernel incl. the MGS cluster and the dense DSTs), C2 apply and K_N apply, C3 at
1024 partitioned ×2 (level-2 exchange kernels), C4 32³ solve (3D path) and a 3D partitioned apply."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2404_15249_b200 import KFBI  # noqa: E402


def solve(prob):
    k = KFBI(prob)
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(prob.n + 1) * prob.h
    G = np.meshgrid(*([x] * prob.dim), indexing="ij")
    f = lambda *a: W.f_exact(prob.kappa, *a)
    u, phi, st = k.solve(W.u_exact(*pz.T), f(*G), f(*pq.T), f(*pz.T))
    torch.cuda.synchronize()
    print(prob.name, prob.n, st, flush=True)


solve(W.C1(64))
k = KFBI(W.C2(256))
print("C2 apply", float(k.apply(W.random_density(k.M, 0)).abs().max()))
kn = KFBI(W.neumann(W.C2(256)))
print("C2 K_N apply", float(kn.apply(W.random_density(kn.M, 0)).abs().max()))
kw = KFBI(W.C3(1024), world=2, rank=-1)
print("C3 x2 apply", float(kw.apply(W.random_density(kw.M, 1)).abs().max()))
solve(W.C4(32))
k3 = KFBI(W.C4(64), world=2, rank=-1)
print("C4 x2 apply", float(k3.apply(W.random_density(k3.M, 2)).abs().max()))
torch.cuda.synchronize()
print("sanitize workload done")
