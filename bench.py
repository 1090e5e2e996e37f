#!/usr/bin/env python
"""KFBI solve benchmark (BASELINE.json metric) — one JSON line on rank 0.

step   = one full kfbi_solve of the workload (volume apply, GMRES(30) on K̃φ = ĝ with one
         interface solve per Arnoldi step, explicit residuals, final field): every row
         A1-A9 of SURVEY §8(a).  Inputs resident in HBM when the timed region starts.
value  = grid points per second per interface solve = U · n_applies / t_step,
         U = (N−1)² unknowns.  Also reported: solve seconds, apply µs.
e2e    = the same metric through the public API with pinned HOST inputs/outputs: the H2D
         copy of g, f (grid, intersections, control points) and the D2H copy of u inside
         the timed region.
cpu_baseline: the CPU oracle (oracle/) as it stands, one full solve of the same workload on all
         host cores (scipy.fft workers; BASELINE.md's CPU plan), rank 0 at N = 1.
--impl reference: the CPU oracle as it stands, one K_D apply of the same workload per step, on
         all host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workloads as W  # noqa: E402

METRIC = "KFBI solve: grid-pts/s per interface solve"
UNIT = "grid-pts/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get("hbm_gbs", 6650.0), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
                self.lines = [l for l in out.splitlines() if l.strip()]
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def make_inputs(k, prob):
    """Manufactured problem u* (reading R24) at the context's own points: g_D = u*|Γ, or for the
    Neumann BVP g_N = n·∇u* with the context's outward normals."""
    n = prob.n
    pz, pq = k.points("ctrl"), k.points("isect")
    x = prob.lo + np.arange(n + 1) * prob.h
    f = lambda *a: W.f_exact(prob.kappa, *a)
    G = np.meshgrid(*([x] * prob.dim), indexing="ij")
    if prob.bc == W.NEUMANN:
        nz = k.points("normal")
        ux, uy = W.grad_u_exact(*pz.T)
        g = ux * nz[:, 0] + uy * nz[:, 1]
    else:
        g = W.u_exact(*pz.T)
    return (g, f(*G).ravel(), f(*pq.T), f(*pz.T))


def host_cpu():
    """Host description for the CPU baselines (nproc, lscpu model and sockets)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for l in out.splitlines():
            k, _, v = l.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:
        pass
    return info


def oracle_workers():
    """The oracle runs as it stands; only its library primitives get the host's cores: scipy.fft's
    worker pool (its DST-I passes) and the BLAS thread pool.  NumPy element-wise work stays serial."""
    import scipy.fft
    return scipy.fft.set_workers(os.cpu_count() or 1)


def cpu_oracle_solve_rate(prob):
    """The oracle's full Dirichlet solve (Y apply, Alg. 5 GMRES, final field) of the
    workload on all host cores, as BASELINE.md plans the CPU column: U × interface solves / seconds."""
    from oracle.bie import Oracle2D
    from oracle.bie3d import Oracle3D
    with oracle_workers():
        t0 = time.perf_counter()
        o = Oracle2D(prob) if prob.dim == 2 else Oracle3D(prob)
        t_setup = time.perf_counter() - t0
        f = lambda *a: W.f_exact(prob.kappa, *a)
        g = W.u_exact(*(o.ctrl_points() if prob.dim == 2 else o.points().T))
        t0 = time.perf_counter()
        _, _, st = o.solve(g, f)
        t = time.perf_counter() - t0
    n_solves = st.n_applies + 2          # + the Y apply and the final field (as kfbi_solve counts)
    return prob.unknowns * n_solves / t, t, t_setup, st


def run_reference(args, prob):
    """The base contract's reference arm for this tier: the CPU oracle as it stands, one K_D apply of
    the workload per step, on all host cores (scipy.fft workers), rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle.bie import Oracle2D
    from oracle.bie3d import Oracle3D
    U = prob.unknowns
    with oracle_workers():
        o = Oracle2D(prob) if prob.dim == 2 else Oracle3D(prob)
        phi = W.random_density(o.M, 0)
        apply = o.apply_K if prob.dim == 2 else o.apply_KD
        for _ in range(args.warmup):
            apply(phi)
        ts = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            apply(phi)
            ts.append(time.perf_counter() - t0)
    t = float(np.mean(ts))
    v = U / t
    cpu = host_cpu()
    sample = (f"one K_D apply (interface solve) of {prob.name} N={prob.n} per step; scipy.fft workers = "
              f"{cpu['nproc']} host cores, NumPy element-wise serial")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": prob.name, "grid": prob.n, "kappa": prob.kappa, "M": o.M},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cpu["nproc"], "kind": "oracle", "sample": sample,
                         "host": cpu},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kfbi", choices=["kfbi", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--n", type=int, default=0, help="override grid size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--method", default="gmres", choices=["gmres", "richardson", "bicgstab"],
                    help="outer iteration (P:495-502 Richardson, BiCGSTAB, GMRES Alg. 5)")
    ap.add_argument("--bc", default="dirichlet", choices=["dirichlet", "neumann"],
                    help="boundary condition (neumann: 2D, κ > 0 configs, e.g. --config C2)")
    args = ap.parse_args()
    prob = W.CONFIGS[args.config](args.n) if args.n else W.CONFIGS[args.config]()
    if args.bc == "neumann":
        prob = W.neumann(prob)
    if args.impl == "reference":
        return run_reference(args, prob)

    import torch
    import torch.distributed as dist

    from paper_2404_15249_b200 import KFBI, broadcast_unique_id, launch_count

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # multi-GPU: slabs along x over NCCL when the world size divides the slab units
    # (2D: level-2 segments, N/512; 3D: ADM blocks, N/16); otherwise independent replicas
    sharded = world > 1 and (prob.n % (512 * world) == 0 if prob.dim == 2 else prob.n % (16 * world) == 0)
    if world > 1 and not sharded:
        # the path shards (slabs of level-2 segments / ADM blocks): N replicas of the whole
        # problem would read as scaling, so a world size that does not divide the slab units is refused
        if rank == 0:
            print(json.dumps({"metric": METRIC, "error": f"world {world} does not divide {prob.name} N={prob.n} into "
                              f"slabs ({'N/512 segments' if prob.dim == 2 else 'N/16 ADM blocks'})"}))
        dist.destroy_process_group()
        raise SystemExit(2)
    if sharded:
        k = KFBI(prob, device=local, world=world, rank=rank, nccl_id=broadcast_unique_id())
    else:
        k = KFBI(prob, device=local)
    g, fgrid, fq, fz = make_inputs(k, prob)
    if sharded:   # one rank per process: f and u are the rank's node slab (kfbi_local_slab)
        fgrid = np.ascontiguousarray(fgrid.reshape((prob.n + 1,) * prob.dim)[k.local_slice()]).reshape(-1)
    t = lambda a: torch.tensor(a, dtype=torch.float64, device=dev)
    g_d, fg_d, fq_d, fz_d = t(g), t(fgrid), t(fq), t(fz)
    u_d = torch.empty(k.local_nodes, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def step():
        return k.solve(g_d, fg_d, fq_d, fz_d, u=u_d, method=args.method)

    for _ in range(args.warmup):
        _, _, st = step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    times, stats = [], None
    l0 = launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()                                   # L2 flush between timed steps
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            _, _, stats = step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    launches = launch_count() - l0
    torch.cuda.synchronize()
    barrier()
    t_step = sum(times) / len(times)
    if world > 1:
        tt = torch.tensor([t_step], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step = float(tt.item())
    U = prob.unknowns
    n_app = stats.n_applies
    copies = 1
    value = copies * U * n_app / t_step

    # e2e through the public API with pinned host buffers.  Single-grid layouts move only the Ω-node
    # values of f and u (kfbi_scatter_omega / kfbi_gather_omega: f is zero-extended off Ω, and
    # u_h is valid on Ω); slab-sharded runs move each rank's node slab of f and u.
    pin = lambda a: torch.tensor(a, dtype=torch.float64).pin_memory()
    compact = not sharded
    omega_io = compact   # kfbi_solve_opts.omega_io (single-context grids)
    if compact:
        omask = k.node_mask().reshape(-1).astype(bool)
        n_out = int(omask.sum())
        fg_h = pin(np.ascontiguousarray(fgrid.reshape(-1)[omask]))
        fg_full = [torch.empty(k.n_nodes, dtype=torch.float64, device=dev) for _ in range(2)]
    else:
        n_out = k.local_nodes
        fg_h = pin(fgrid)
    g_h, fq_h, fz_h = pin(g), pin(fq), pin(fz)
    u_h = torch.empty(n_out, dtype=torch.float64).pin_memory()
    u_c = torch.empty(n_out, dtype=torch.float64, device=dev) if compact else None

    def solve_io(gd, fgd, fqd, fzd, b, u=None, async_final=False):
        """kfbi_solve on device inputs; with compact transfers f is scattered first and the Ω values
        of u gathered after; returns the device array the host copy reads.  async_final: the solve
        returns with its final field still running on the stream (the serving loop's next host work
        overlaps it; every later use is stream-ordered)."""
        if compact and omega_io:   # the solve reads f and writes u as Ω-node values itself
            u, _, st_ = k.solve(gd, fgd, fqd, fzd, u=u_c if b is None else u_cs[b], method=args.method,
                                async_final=async_final, omega_io=True)
            return u
        if compact:
            u, _, st_ = k.solve(gd, k.scatter_omega(fgd, grid=fg_full[b]), fqd, fzd, u=u, method=args.method,
                                async_final=async_final)
            return k.gather_omega(u, compact=u_c if b is None else u_cs[b])
        u, _, st_ = k.solve(gd, fgd, fqd, fzd, u=u, method=args.method, async_final=async_final)
        return u.view(-1)

    u_cs = [torch.empty(n_out, dtype=torch.float64, device=dev) for _ in range(2)] if compact else None
    e2e_t = []
    for it in range(args.warmup + args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        gd = g_h.to(dev, non_blocking=True)
        fgd = fg_h.to(dev, non_blocking=True)
        fqd = fq_h.to(dev, non_blocking=True)
        fzd = fz_h.to(dev, non_blocking=True)
        uo = solve_io(gd, fgd, fqd, fzd, 0)
        u_h.copy_(uo, non_blocking=True)
        e1.record(stream)
        e1.synchronize()
        if it >= args.warmup:
            e2e_t.append(e0.elapsed_time(e1) / 1e3)
    t_e2e = sum(e2e_t) / len(e2e_t)
    if world > 1:
        tt = torch.tensor([t_e2e], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e = float(tt.item())
    h2d = 8 * (g.size + fg_h.numel() + fq.size + fz.size)
    d2h = 8 * n_out

    # e2e, pipelined serving loop through the same public API: step k+1's inputs are uploaded on an
    # H2D copy stream while step k solves, and step k's field is downloaded on a D2H copy stream while
    # step k+1 solves (double-buffered device inputs/outputs; PCIe is full duplex).  Every step still
    # moves its own inputs and result; the timed region spans the first upload to the last download.
    def e2e_pipelined(nsteps):
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        din = [[torch.empty_like(x, device=dev) for x in (g_h, fg_h, fq_h, fz_h)] for _ in range(2)]
        dout = [torch.empty(k.local_nodes, dtype=torch.float64, device=dev) for _ in range(2)]
        hout = [torch.empty(n_out, dtype=torch.float64).pin_memory() for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]

        def upload(j):
            b = j % 2
            with torch.cuda.stream(h2d_s):
                if j >= 2:
                    h2d_s.wait_event(ev_done[b])            # solve j−2 no longer reads these inputs
                for dst, src in zip(din[b], (g_h, fg_h, fq_h, fz_h)):
                    dst.copy_(src, non_blocking=True)
                ev_in[b].record(h2d_s)

        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        torch.cuda.synchronize()
        t0.record(h2d_s)
        upload(0)
        for j in range(nsteps):
            b = j % 2
            if j + 1 < nsteps:
                upload(j + 1)
            stream.wait_event(ev_in[b])
            if j >= 2:
                stream.wait_event(ev_out[b])                # download j−2 has left dout[b]
            uo = solve_io(*din[b], b, u=dout[b], async_final=True)
            ev_done[b].record(stream)
            with torch.cuda.stream(d2h_s):
                d2h_s.wait_event(ev_done[b])
                hout[b].copy_(uo, non_blocking=True)
                ev_out[b].record(d2h_s)
        d2h_s.wait_stream(h2d_s)
        t1.record(d2h_s)
        t1.synchronize()
        return t0.elapsed_time(t1) / 1e3 / nsteps

    # the pipelined loop's fill and drain (one upload, one download: ≈ 7.5 ms at C3) are amortised over at
    # least 30 steps so that s_per_step is the serving loop's steady state (the step count is reported)
    n_e2e = max(args.steps, 30)
    e2e_pipelined(max(args.warmup, 2))
    t_e2e_pipe = e2e_pipelined(n_e2e)
    if world > 1:
        tt = torch.tensor([t_e2e_pipe], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_e2e_pipe = float(tt.item())

    # per-kernel device times of the K_D apply (CUDA events on the launching stream)
    phi = torch.tensor(W.random_density(k.M, 0), device=dev)
    prof = k.profile_apply(phi, reps=20)
    model = k.apply_model()
    peak, peak_src = measured_peaks()
    cand = {"sweep": model["bytes_sweep"], "inverse": model["bytes_inverse"]}
    dom = max(cand, key=lambda n: prof[n])
    achieved = cand[dom] / (prof[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": f"k_{dom}", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": cand[dom],
                "share_of_apply": prof[dom] / prof["apply"],
                "kernel_ms": {n: round(v, 4) for n, v in prof.items()}}
    ncu_csv = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu_csv):
        try:
            roofline["traffic"] = json.load(open(ncu_csv)).get(f"{prob.name}:{prob.n}:k_{dom}")
        except Exception:
            pass
    # the FP64 side of the same kernels: ncu's executed FP64 FLOPs per launch (2·DFMA + DADD + DMUL,
    # profiles/ncu_fp64.json) over the live CUDA-event time, against the measured FP64 peak
    # (profiles/fp64_peak.json, tools/fp64_peak.cu)
    try:
        fl = json.load(open(os.path.join(ROOT, "profiles", "ncu_fp64.json")))
        pk = json.load(open(os.path.join(ROOT, "profiles", "fp64_peak.json")))["fp64_tflops"]
        fp = {}
        for n in ("sweep", "inverse"):
            f = fl.get(f"{prob.name}:{prob.n}:k_{n}")
            if f:
                a = f / (prof[n] * 1e-3) / 1e12
                fp[f"k_{n}"] = {"achieved": a, "peak": pk, "unit": "TFLOP/s", "frac": a / pk, "flops_per_launch": f}
        if fp:
            roofline["fp64"] = fp
    except Exception:
        pass

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_step, "higher_is_better": True,
        "scaling": "strong" if sharded else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (manufactured u*, reading R24)",
        "config": {"workload": prob.name, "grid": prob.n, "unknowns": U, "kappa": prob.kappa, "M": k.M,
                   "bc": "neumann" if prob.bc == W.NEUMANN else "dirichlet", "method": args.method,
                   "intersections": k.nq, "irregular": k.nirr,
                   "parallelism": "single-gpu" if world == 1 else (f"slabs{world}-nccl" if sharded else f"replicas{world}"),
                   "l2": "flushed between timed steps (256 MB write before each step)"},
        "solve_s": t_step, "gmres_iters": stats.iters, "n_applies": n_app, "rel_residual": stats.rel_residual,
        "apply_us": 1e3 * prof["apply"], "apply_grid_pts_per_s": U / (prof["apply"] * 1e-3),
        "e2e": {"value": copies * U * n_app / t_e2e_pipe, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "s_per_step": t_e2e_pipe, "steps": n_e2e,
                "mode": "pipelined serving loop: H2D of step k+1 and D2H of step k overlap the solves "
                        "(two copy streams, double-buffered); timed from the first upload to the last download"
                        + ("; f and u cross PCIe as their Omega-node values, which kfbi_solve reads and writes "
                           "directly (opts.omega_io)" if omega_io else
                           "; f and u cross PCIe as their Omega-node values (kfbi_scatter_omega before and "
                           "kfbi_gather_omega after each solve, inside the timed region)" if compact else ""),
                "serial": {"value": copies * U * n_app / t_e2e, "s_per_step": t_e2e,
                           "mode": "H2D, solve, D2H back to back every step"}},
        "gpu_launches": launches, "gpu_launches_per_step": launches / args.steps,
        "roofline": roofline,
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, t, t_setup, st = cpu_oracle_solve_rate(prob)
        cpu = host_cpu()
        line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": cpu["nproc"], "kind": "oracle",
                                "sample": f"one full oracle solve of {prob.name} N={prob.n} ({t:.1f} s, "
                                          f"{st.iters} GMRES iterations, {st.n_applies + 2} interface solves; "
                                          f"setup {t_setup:.0f} s untimed); scipy.fft workers = {cpu['nproc']} "
                                          f"host cores, NumPy element-wise serial",
                                "host": cpu, "solve_s": t, "gpu_speedup_solve": t / t_step}
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
