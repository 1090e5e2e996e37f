"""Thin ctypes binding of include/kfbi.h (argument marshalling only).

Every step of the KFBI path runs in the sm_100a kernels of lib/libkfbi.so; PyTorch only
provides device memory (the workspace and I/O tensors) and the CUDA stream.  There is no
CPU fallback: if the library is missing this module raises.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libkfbi.so")

OK, EINVAL, EGEOM, ENOCONV, ECUDA, ENCCL, ENOMEM, EUNSUPPORTED, EBREAKDOWN = range(9)
_NAMES = {0: "OK", 1: "EINVAL", 2: "EGEOM", 3: "ENOCONV", 4: "ECUDA", 5: "ENCCL", 6: "ENOMEM", 7: "EUNSUPPORTED",
          8: "EBREAKDOWN"}

EXPORTS = ["kfbi_version", "kfbi_last_error", "kfbi_last_setup_error", "kfbi_get_unique_id", "kfbi_setup",
           "kfbi_workspace_size", "kfbi_set_workspace", "kfbi_sizes", "kfbi_points", "kfbi_node_mask",
           "kfbi_apply", "kfbi_solve", "kfbi_apply_model", "kfbi_destroy", "kfbi_test_fast_solve",
           "kfbi_test_interface_solve", "kfbi_test_setup_dump", "kfbi_profile_apply", "kfbi_launch_count",
           "kfbi_slab", "kfbi_gray_scott_step", "kfbi_setup_scratch_size", "kfbi_setup_device",
           "kfbi_omega_count", "kfbi_scatter_omega", "kfbi_gather_omega", "kfbi_local_slab",
           "kfbi_node_mask_device"]


class KfbiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"kfbi {_NAMES.get(code, code)}: {msg}")
        self.code = code


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("lo", C.c_double * 3), ("hi", C.c_double * 3), ("n", C.c_int32 * 3)]


class Component(C.Structure):
    _fields_ = [("kind", C.c_int32), ("role", C.c_int32), ("center", C.c_double * 3), ("p", C.c_double * 4),
                ("n_ctrl", C.c_int32)]


class Boundary(C.Structure):
    _fields_ = [("ncomp", C.c_int32), ("comp", C.POINTER(Component))]


class Pde(C.Structure):
    _fields_ = [("kappa", C.c_double), ("bc", C.c_int32)]


class Dist(C.Structure):
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("device", C.c_int32), ("nccl_id", C.c_void_p)]


class SolveOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("restart", C.c_int32), ("max_restarts", C.c_int32),
                ("method", C.c_int32), ("gamma", C.c_double), ("async_final", C.c_int32), ("omega_io", C.c_int32)]


METHODS = {"gmres": 0, "richardson": 1, "bicgstab": 2}


class SolveStats(C.Structure):
    _fields_ = [("iters", C.c_int32), ("restarts", C.c_int32), ("n_applies", C.c_int32), ("converged", C.c_int32),
                ("rel_residual", C.c_double), ("t_solve_s", C.c_double)]


_lib = None


def load(path: str = LIB_PATH):
    """Load lib/libkfbi.so (raises if it is not built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA library {path} is not built; run python -m paper_2404_15249_b200.build")
    lib = C.CDLL(path)
    vp, dp, i32, i64p = C.c_void_p, C.POINTER(C.c_double), C.c_int32, C.POINTER(C.c_int64)
    lib.kfbi_version.restype = C.c_char_p
    lib.kfbi_last_error.restype = C.c_char_p
    lib.kfbi_last_error.argtypes = [vp]
    lib.kfbi_last_setup_error.restype = C.c_char_p
    lib.kfbi_get_unique_id.argtypes = [vp]
    lib.kfbi_setup.argtypes = [C.POINTER(Grid), C.POINTER(Boundary), C.POINTER(Pde), C.POINTER(Dist), vp, C.POINTER(vp)]
    lib.kfbi_omega_count.argtypes = [vp, i64p]
    lib.kfbi_scatter_omega.argtypes = [vp, vp, vp, vp]
    lib.kfbi_gather_omega.argtypes = [vp, vp, vp, vp]
    lib.kfbi_setup_scratch_size.argtypes = [C.POINTER(Grid), C.POINTER(C.c_size_t)]
    lib.kfbi_setup_device.argtypes = [C.POINTER(Grid), C.POINTER(Boundary), C.POINTER(Pde), C.POINTER(Dist), vp, vp,
                                      C.c_size_t, C.POINTER(vp)]
    lib.kfbi_workspace_size.argtypes = [vp, C.POINTER(C.c_size_t)]
    lib.kfbi_set_workspace.argtypes = [vp, vp, C.c_size_t]
    lib.kfbi_sizes.argtypes = [vp, i64p, i64p, i64p, i64p]
    lib.kfbi_local_slab.argtypes = [vp, i64p, i64p]
    lib.kfbi_points.argtypes = [vp, i32, dp]
    lib.kfbi_node_mask.argtypes = [vp, C.POINTER(C.c_int8)]
    lib.kfbi_node_mask_device.argtypes = [vp, vp, vp]
    lib.kfbi_apply.argtypes = [vp, vp, vp, vp]
    lib.kfbi_solve.argtypes = [vp, vp, vp, vp, vp, vp, vp, vp, C.POINTER(SolveOpts), C.POINTER(SolveStats), vp]
    lib.kfbi_apply_model.argtypes = [vp, dp, dp, dp]
    lib.kfbi_destroy.argtypes = [vp]
    lib.kfbi_test_fast_solve.argtypes = [vp, vp, vp, vp]
    lib.kfbi_test_interface_solve.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    lib.kfbi_test_setup_dump.argtypes = [vp, i32, i64p]
    lib.kfbi_profile_apply.argtypes = [vp, vp, vp, i32, dp, vp]
    lib.kfbi_launch_count.argtypes = [i64p]
    lib.kfbi_slab.argtypes = [vp, i32, i64p]
    lib.kfbi_gray_scott_step.argtypes = [vp, vp, vp, vp, vp, vp, i32, vp, C.c_double, dp, C.c_double,
                                         C.POINTER(C.c_int32), vp]
    for name in EXPORTS:
        getattr(lib, name).restype = C.c_char_p if name in ("kfbi_version", "kfbi_last_error",
                                                            "kfbi_last_setup_error") else C.c_int32
    _lib = lib
    return lib


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 of a multi-GPU run)."""
    buf = (C.c_uint8 * 128)()
    lib = load()
    st = lib.kfbi_get_unique_id(buf)
    if st != OK:
        raise KfbiError(st, lib.kfbi_last_setup_error().decode())
    return bytes(buf)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 creates the NCCL id; torch.distributed broadcasts it as a uint8[128] tensor."""
    import torch
    import torch.distributed as dist
    t = torch.zeros(128, dtype=torch.uint8)
    if dist.get_rank(group) == 0:
        t.copy_(torch.frombuffer(bytearray(unique_id()), dtype=torch.uint8))
    if dist.get_backend(group) == "nccl":
        d = t.cuda()
        dist.broadcast(d, 0, group=group)
        t = d.cpu()
    else:
        dist.broadcast(t, 0, group=group)
    return bytes(t.tolist())


def launch_count() -> int:
    c = C.c_int64()
    load().kfbi_launch_count(C.byref(c))
    return c.value


@dataclasses.dataclass
class Stats:
    iters: int
    restarts: int
    n_applies: int
    converged: bool
    rel_residual: float
    t_solve_s: float


class KFBI:
    """One context per (problem, device).  `problem` is any object with dim, n, lo, hi,
    kappa and comps (each with kind, role, center, p, n_ctrl) — e.g. workloads.Problem."""

    def __init__(self, problem, device: int = 0, stream=None, workspace: bool = True, world: int = 1,
                 rank: int = 0, nccl_id: bytes = None, device_setup: bool = False):
        """world > 1: slab `rank` of a multi-GPU run (nccl_id from broadcast_unique_id), or
        rank = −1 to run all slabs in this process (single-GPU emulation of the partition).
        device_setup: run the O(N²) phases of Procedure 1 on the GPU (kfbi_setup_device, 2D)."""
        import torch
        self.torch = torch
        self.lib = load()
        self.device = torch.device("cuda", device)
        self.ctx = None
        self.problem = problem
        d = problem.dim
        g = Grid(d, (C.c_double * 3)(*([problem.lo] * 3)), (C.c_double * 3)(*([problem.hi] * 3)),
                 (C.c_int32 * 3)(*([problem.n] * 3)))
        comps = (Component * len(problem.comps))()
        for k, c in enumerate(problem.comps):
            cen = list(c.center) + [0.0] * (3 - len(c.center))
            comps[k] = Component(c.kind, c.role, (C.c_double * 3)(*cen), (C.c_double * 4)(*c.p), c.n_ctrl)
        self._comps = comps
        b = Boundary(len(problem.comps), comps)
        pde = Pde(problem.kappa, int(getattr(problem, "bc", 0)))
        self._nccl = (C.c_uint8 * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        dist = Dist(world, rank, device, C.cast(self._nccl, C.c_void_p) if self._nccl is not None else None)
        self.world, self.rank = world, rank
        ctx = C.c_void_p()
        if device_setup:
            sb = C.c_size_t()
            st = self.lib.kfbi_setup_scratch_size(C.byref(g), C.byref(sb))
            if st != OK:
                raise KfbiError(st, self.lib.kfbi_last_setup_error().decode())
            scratch = torch.empty(sb.value, dtype=torch.uint8, device=self.device)
            with torch.cuda.device(self.device):
                strm = torch.cuda.current_stream(self.device).cuda_stream
                st = self.lib.kfbi_setup_device(C.byref(g), C.byref(b), C.byref(pde), C.byref(dist), C.c_void_p(strm),
                                                C.c_void_p(scratch.data_ptr()), sb.value, C.byref(ctx))
            del scratch
        else:
            st = self.lib.kfbi_setup(C.byref(g), C.byref(b), C.byref(pde), C.byref(dist), None, C.byref(ctx))
        if st != OK:
            raise KfbiError(st, self.lib.kfbi_last_setup_error().decode())
        self.ctx = ctx
        nb = C.c_size_t()
        self._check(self.lib.kfbi_workspace_size(ctx, C.byref(nb)))
        self.workspace_bytes = nb.value
        if workspace:   # host-only setups (CPU tests of Procedure 1) skip the device part
            self.ws = torch.empty(nb.value, dtype=torch.uint8, device=self.device)
            with torch.cuda.device(self.device):
                self._check(self.lib.kfbi_set_workspace(ctx, C.c_void_p(self.ws.data_ptr()), nb.value))
        M, nq, nirr, nn = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.kfbi_sizes(ctx, C.byref(M), C.byref(nq), C.byref(nirr), C.byref(nn)))
        self.M, self.nq, self.nirr, self.n_nodes = M.value, nq.value, nirr.value, nn.value
        self.n = problem.n
        shp, off = (C.c_int64 * 3)(), (C.c_int64 * 3)()
        self._check(self.lib.kfbi_local_slab(ctx, shp, off))
        d = problem.dim
        self.local_shape = tuple(shp[:d])          # f and u of kfbi_solve (the full grid unless one
        self.local_offset = tuple(off[:d])         # rank per process, see include/kfbi.h)
        self.local_nodes = int(np.prod(self.local_shape))

    # ------------------------------------------------------------------ helpers
    def _check(self, st):
        if st != OK:
            raise KfbiError(st, self.lib.kfbi_last_error(self.ctx).decode())

    def _stream(self, stream):
        """cudaStream_t for a call.  Inputs are converted on torch's current stream, so an explicit
        other stream first waits on it (no read of a half-copied input)."""
        cur = self.torch.cuda.current_stream(self.device)
        if stream is not None and stream != cur:
            stream.wait_stream(cur)
        return C.c_void_p((stream if stream is not None else cur).cuda_stream)

    def _keep(self, stream, *tensors):
        """Tensors read or written by work still queued on an explicit non-current stream stay
        allocated until that work is done (caching-allocator record_stream)."""
        if stream is None or stream == self.torch.cuda.current_stream(self.device):
            return
        for x in tensors:
            if x is not None:
                x.record_stream(stream)

    def _out(self, x, n, name):
        """A caller-supplied output buffer: float64, contiguous, on the context's device, n values."""
        t = self.torch
        if (not isinstance(x, t.Tensor) or x.dtype != t.float64 or x.device != self.device
                or not x.is_contiguous() or x.numel() != n):
            raise ValueError(f"{name} must be a contiguous float64 tensor of {n} values on {self.device}")
        return x

    def _dev(self, x, n=None):
        t = self.torch
        if x is None:
            return None
        if not isinstance(x, t.Tensor):
            x = t.as_tensor(np.ascontiguousarray(x, dtype=np.float64))
        x = x.to(device=self.device, dtype=t.float64).contiguous()
        if n is not None and x.numel() != n:
            raise ValueError(f"expected {n} values, got {x.numel()}")
        return x

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.kfbi_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ API
    def points(self, which="ctrl"):
        """which: "ctrl" (control points), "isect" (intersection nodes), "normal" (outward unit
        normals at the control points)."""
        code = {"ctrl": 0, "isect": 1, "normal": 2}[which]
        n = self.nq if which == "isect" else self.M
        out = np.zeros((n, self.problem.dim))
        self._check(self.lib.kfbi_points(self.ctx, code, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def omega_count(self):
        n = C.c_int64()
        self._check(self.lib.kfbi_omega_count(self.ctx, C.byref(n)))
        return n.value

    def scatter_omega(self, compact, grid=None, stream=None):
        """Full (N+1)^d grid from the Ω-node values (0 off Ω) — kfbi_scatter_omega."""
        t = self.torch
        compact = self._out(compact, self.omega_count(), "compact")
        grid = (t.empty(self.n_nodes, dtype=t.float64, device=self.device) if grid is None
                else self._out(grid, self.n_nodes, "grid"))
        with t.cuda.device(self.device):
            self._check(self.lib.kfbi_scatter_omega(self.ctx, _ptr(compact), _ptr(grid), self._stream(stream)))
        self._keep(stream, compact, grid)
        return grid

    def gather_omega(self, grid, compact=None, stream=None):
        """Ω-node values of a full grid — kfbi_gather_omega."""
        t = self.torch
        grid = self._out(grid.reshape(-1) if grid.is_contiguous() else grid, self.n_nodes, "grid")
        compact = (t.empty(self.omega_count(), dtype=t.float64, device=self.device) if compact is None
                   else self._out(compact, self.omega_count(), "compact"))
        with t.cuda.device(self.device):
            self._check(self.lib.kfbi_gather_omega(self.ctx, _ptr(grid), _ptr(compact), self._stream(stream)))
        self._keep(stream, grid, compact)
        return compact

    def node_mask_device(self, stream=None):
        """Ω mask of this context's node slab as a device int8 tensor (kfbi_node_mask_device)."""
        t = self.torch
        out = t.empty(self.local_nodes, dtype=t.int8, device=self.device)
        with t.cuda.device(self.device):
            self._check(self.lib.kfbi_node_mask_device(self.ctx, _ptr(out), self._stream(stream)))
        self._keep(stream, out)
        return out.view(self.local_shape)

    def node_mask(self):
        out = np.zeros(self.n_nodes, dtype=np.int8)
        self._check(self.lib.kfbi_node_mask(self.ctx, out.ctypes.data_as(C.POINTER(C.c_int8))))
        return out.reshape((self.n + 1,) * self.problem.dim)

    def apply(self, phi, out=None, stream=None):
        phi = self._dev(phi, self.M)
        out = self.torch.empty_like(phi) if out is None else self._out(out, self.M, "out")
        with self.torch.cuda.device(self.device):
            self._check(self.lib.kfbi_apply(self.ctx, _ptr(phi), _ptr(out), self._stream(stream)))
        self._keep(stream, phi, out)
        return out

    def solve(self, g, f_grid=None, f_isect=None, f_ctrl=None, phi0=None, tol=1e-8, restart=30,
              max_restarts=50, u=None, stream=None, raise_on_noconv=True, method="gmres", gamma=1.0,
              async_final=False, omega_io=False):
        """omega_io: f_grid and u hold the Ω-node values only (omega_count() entries, row-major node
        order; single-context grids) and u is returned flat in that layout."""
        t = self.torch
        nf = self.omega_count() if omega_io else self.local_nodes
        g = self._dev(g, self.M)
        fg = self._dev(f_grid, nf)
        fq = self._dev(f_isect, self.nq)
        fz = self._dev(f_ctrl, self.M)
        p0 = self._dev(phi0, self.M)
        u = (t.empty(nf, dtype=t.float64, device=self.device) if u is None
             else self._out(u.reshape(-1) if isinstance(u, t.Tensor) and u.is_contiguous() else u, nf, "u"))
        phi = t.empty(self.M, dtype=t.float64, device=self.device)
        opts = SolveOpts(tol, restart, max_restarts, METHODS[method], gamma, 1 if async_final else 0,
                         1 if omega_io else 0)
        st = SolveStats()
        with t.cuda.device(self.device):
            code = self.lib.kfbi_solve(self.ctx, _ptr(g), _ptr(fg), _ptr(fq), _ptr(fz), _ptr(p0), _ptr(u), _ptr(phi),
                                       C.byref(opts), C.byref(st), self._stream(stream))
        self._keep(stream, g, fg, fq, fz, p0, u, phi)
        if code != OK and (code != ENOCONV or raise_on_noconv):
            self._check(code)
        stats = Stats(st.iters, st.restarts, st.n_applies, bool(st.converged), st.rel_residual, st.t_solve_s)
        return (u if omega_io else u.view(self.local_shape)), phi, stats

    def local_slice(self):
        """numpy index of this context's node slab in the full grid (f and u of solve())."""
        return tuple(slice(o, o + n) for o, n in zip(self.local_offset, self.local_shape))

    def slab(self, rank=None):
        out = (C.c_int64 * 6)()
        self._check(self.lib.kfbi_slab(self.ctx, self.rank if rank is None else rank, out))
        keys = (["g_lo", "g_hi", "col_lo", "col_hi", "o_lo", "o_hi"] if self.problem.dim == 2
                else ["b_lo", "b_hi", "i_lo", "i_hi", "w_lo", "w_hi"])
        return dict(zip(keys, list(out)))

    def apply_model(self):
        a, b, c = C.c_double(), C.c_double(), C.c_double()
        self._check(self.lib.kfbi_apply_model(self.ctx, C.byref(a), C.byref(b), C.byref(c)))
        return {"bytes_sweep": a.value, "bytes_inverse": b.value, "unknowns": c.value}

    def profile_apply(self, phi, reps=10, stream=None):
        """Per-kernel CUDA-event times (ms) of one apply.  2D: spline, correct, sweep (sparse forward
        DST fused with the block tridiagonal solves), reduced, inverse, hole, interp, total; 3D: lsq,
        correct, sweep (sparse forward DST k_fwd3s), tridiag (+ reduced), inverse (k_inv3y), zeval,
        interp, total."""
        phi = self._dev(phi, self.M)
        out = self.torch.empty_like(phi)
        ms = (C.c_double * 8)()
        self._check(self.lib.kfbi_profile_apply(self.ctx, _ptr(phi), _ptr(out), reps, ms, self._stream(stream)))
        names = (["spline", "correct", "sweep", "reduced", "inverse", "hole", "interp", "apply"] if self.problem.dim == 2
                 else ["lsq", "correct", "sweep", "tridiag", "inverse", "zeval", "interp", "apply"])
        return dict(zip(names, list(ms)))

    # ------------------------------------------------------------------ test-only
    def test_fast_solve(self, rhs_full, stream=None):
        rhs = self._dev(rhs_full, self.n_nodes)
        v = self.torch.empty_like(rhs)
        self._check(self.lib.kfbi_test_fast_solve(self.ctx, _ptr(rhs), _ptr(v), self._stream(stream)))
        return v.view((self.n + 1,) * self.problem.dim)

    def test_interface_solve(self, base_full, jq, jz, want_field=True, stream=None):
        base = self._dev(base_full, self.n_nodes)
        ncol = 6 if self.problem.dim == 2 else 10
        jq = self._dev(jq, self.nq * ncol)
        jz = self._dev(jz, self.M * ncol)
        v = self.torch.empty(self.n_nodes, dtype=self.torch.float64, device=self.device) if want_field else None
        vp = self.torch.empty(self.M, dtype=self.torch.float64, device=self.device)
        self._check(self.lib.kfbi_test_interface_solve(self.ctx, _ptr(base), _ptr(jq), _ptr(jz), _ptr(v), _ptr(vp),
                                                       self._stream(stream)))
        return (v.view((self.n + 1,) * self.problem.dim) if v is not None else None), vp

    def setup_dump(self, which):
        d = self.problem.dim
        shape = {0: (self.nirr, d), 1: (self.nq, d + 1), 2: (self.M, 6 if d == 2 else 10, d)}[which]
        out = np.zeros(int(np.prod(shape)), dtype=np.int64)
        self._check(self.lib.kfbi_test_setup_dump(self.ctx, which, out.ctypes.data_as(C.POINTER(C.c_int64))))
        return out.reshape(shape)
