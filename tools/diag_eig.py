import numpy as np
import workloads as W
from paper_2404_15249_b200 import KFBI
for n, p, q in [(1024, 3, 501), (2048, 3, 1001), (4096, 3, 2001), (8192, 3, 4001), (8192, 3, 5), (8192, 4001, 3), (8192, 100, 200)]:
    prob = W.problem(f"box{n}", 2, n, [W.ellipse(1.0, 0.8)], 0.0)
    k = KFBI(prob)
    h = prob.h
    i = np.arange(n + 1)
    S = np.outer(np.sin(np.pi * p * i / n), np.sin(np.pi * q * i / n))
    lam = -4 / h ** 2 * (np.sin(np.pi * p / (2 * n)) ** 2 + np.sin(np.pi * q / (2 * n)) ** 2)
    v = k.test_fast_solve(lam * S).cpu().numpy()
    d = np.abs(v - S)
    a, b = np.unravel_index(d.argmax(), d.shape)
    rows = d.max(axis=1)
    print(n, p, q, "max", d.max(), "at", a, b, "a%16", a % 16, "worst rows", np.argsort(rows)[-5:], flush=True)
