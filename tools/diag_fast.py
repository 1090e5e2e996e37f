import numpy as np, workloads as W
from oracle import fastsolve
from paper_2404_15249_b200 import KFBI
for n, kap in [(1024, 0.0), (2048, 0.0), (2048, 1.0)]:
    prob = W.problem(f"box{n}", 2, n, [W.ellipse(1.0, 0.8)], kap)
    k = KFBI(prob)
    rhs = np.random.default_rng(n).uniform(-1, 1, (n + 1, n + 1))
    v = k.test_fast_solve(rhs).cpu().numpy()[1:n, 1:n]
    ref = fastsolve.solve2d(rhs[1:n, 1:n], prob.h, kap)
    for name, x in (("gpu", v), ("oracle", ref)):
        res = fastsolve.apply_operator2d(x, prob.h, kap) - rhs[1:n, 1:n]
        i, j = np.unravel_index(np.abs(res).argmax(), res.shape)
        rowmax = np.abs(res).max(axis=1)
        print(n, kap, name, "res max", np.abs(res).max(), "at", i + 1, j + 1, "(i%16=", (i + 1) % 16, ")",
              "median rowmax", np.median(rowmax), "sep rows max", rowmax[15::16].max(), "nonsep", np.delete(rowmax, np.s_[15::16]).max())
    d = np.abs(v - ref)
    i, j = np.unravel_index(d.argmax(), d.shape)
    print("  diff", d.max() / np.abs(ref).max(), "at", i + 1, j + 1)
