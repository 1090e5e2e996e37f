"""Gray–Scott reaction–diffusion driver: two Neumann contexts and
`kfbi_gray_scott_step` — the reaction, the diffusion sources, the solves and the Crank–Nicolson
update all run in the library; this class only holds the device buffers (marshalling)."""
from __future__ import annotations

import ctypes as C

import numpy as np

from .kfbi import KFBI, _ptr, load


class GrayScott:
    def __init__(self, n, dt, params, problem_fn, initial_fn, tol=1e-8, device=0):
        import torch
        self.torch = torch
        self.dt, self.tol = float(dt), float(tol)
        self.params = (C.c_double * 5)(params["gamma"], params["kr"], params["eps0"], params["eps1"], params["eps2"])
        self.ku = KFBI(problem_fn(n, params["eps1"], dt), device)
        self.kv = KFBI(problem_fn(n, params["eps2"], dt), device)
        prob = self.ku.problem
        x = prob.lo + np.arange(prob.n + 1) * prob.h
        X, Y = np.meshgrid(x, x, indexing="ij")
        u0, v0 = initial_fn(X, Y)
        dev = self.ku.device
        f64 = torch.float64
        self.u = torch.tensor(u0.ravel(), dtype=f64, device=dev)
        self.v = torch.tensor(v0.ravel(), dtype=f64, device=dev)
        self.psi_u = torch.zeros(self.ku.M, dtype=f64, device=dev)
        self.psi_v = torch.zeros(self.kv.M, dtype=f64, device=dev)
        nn = (prob.n + 1) ** 2
        self.scratch = torch.empty(2 * nn + self.ku.nq + 2 * self.ku.M, dtype=f64, device=dev)
        self.warm = 0
        self.iters = []
        self.lib = load()

    def step(self, stream=None):
        it = (C.c_int32 * 2)()
        s = stream if stream is not None else self.torch.cuda.current_stream(self.ku.device)
        code = self.lib.kfbi_gray_scott_step(self.ku.ctx, self.kv.ctx, _ptr(self.u), _ptr(self.v), _ptr(self.psi_u),
                                             _ptr(self.psi_v), self.warm, _ptr(self.scratch), C.c_double(self.dt),
                                             self.params, C.c_double(self.tol), it, C.c_void_p(s.cuda_stream))
        self.ku._check(code)
        self.warm = 1
        self.iters.append((it[0], it[1]))

    def fields(self):
        n = self.ku.problem.n
        return self.u.view(n + 1, n + 1), self.v.view(n + 1, n + 1)
