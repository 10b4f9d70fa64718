#!/usr/bin/env python
"""Benchmark: HVP GDOF/s and implicit-step time of the MPM Lite hot path on B200 (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

A *step* is one full implicit time step of the workload: bin + sort,
P2Q + stretch, C2N, Newton (linearise, Jacobi-PCG with the matrix-free HVP, line search), G2P.
`value` = HVP GDOF/s = 3 * free nodes * HVP launches / summed HVP device time (CUDA events on the
library stream) over the K timed steps.  With N > 1 GPUs the grid is slab-decomposed:
free nodes are summed over ranks (a shared node counts once), the HVP time includes its interface
halo sum and p.Hp allreduce and is the max over ranks.  `ms_per_step` = implicit-step time (device
clock, max over ranks).  Inputs are resident in HBM when the timed region starts; the
HVP's tangent stream (>= 392 MB at cfg4) is larger than the 126 MB L2.

--impl reference times the CPU oracle (oracle/, plain fp64 C, OpenMP colour loops on all host cores) on a
bounded window of the same workload; it is the deliberately slow baseline, not a target.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
KC_REALS = 24  # reals per quadrature point of the compressed tangent (mpl_common.cuh KC_REALS)
sys.path.insert(0, ROOT)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            for nm, val in zip(names, s[3:7]):
                if val.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def hvp_bytes(n_cells, n_nodes, s=4):
    """Algorithmic bytes of one HVP: the 45-number tangent per quadrature point plus
    u (3), Hu (3) and m (1) per active node."""
    return n_cells * 45 * s + n_nodes * 7 * s


def hvp_kernel_name(precision: int = 32) -> str:
    """The HVP kernel the library runs: fp32 k_hvp_wz (MPL_HVP_KERNEL=wh: k_hvp_wh<float, 5>), fp64
    k_hvp_wh<double, 3>."""
    if precision == 64:
        return "k_hvp_wh<double, 3>"
    return "k_hvp_wh<float, 5>" if os.environ.get("MPL_HVP_KERNEL", "wz").startswith("wh") else "k_hvp_wz"


def workload_name(sc) -> str:
    return f"{sc.name}: {sc.n[0]}^3 grid, {sc.n_particles} particles, {len(sc.materials)} material(s), dt={sc.dt}"


def load_traffic(config: str, kernel: str):
    """ncu DRAM bytes (read + write) of one HVP launch of `kernel` on `config` (profiles/hvp_traffic.json,
    from the latest `ncu --set full` capture), else None."""
    p = os.path.join(ROOT, "profiles", "hvp_traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        if d.get("kernel") == kernel:
            return d.get(config)
    return None


# ------------------------------------------------------------------------------------------------
def run_ours(args):
    import torch

    from paper_2602_07853_b200 import dist as pdist
    from paper_2602_07853_b200 import mpl, scenes

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        # NCCL communicator set-up lines (ranks, NVLink / NVLS paths) on stderr, for the run's record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sc = scenes.by_name(args.config, args.precision)
    sel = None
    solver = sc.solver
    stream = torch.cuda.Stream(device=local)
    mode = "1 GPU"
    if ws > 1:
        # slab decomposition: rank r owns the x-slab [cuts[r], cuts[r+1]) of 4-cell blocks; the library's
        # own NCCL communicator carries the halo sums, PCG allreduces and particle migration.  A failure
        # on any rank raises (non-zero exit): there is no silent fallback to replicas.
        nccl_id = pdist.share_nccl_id()
        cuts = pdist.agree_cuts(mpl.slab_cuts(sc, ws))
        ctx = mpl.from_scene_rank(sc, rank, ws, cuts, device=local, nccl_id=nccl_id)
        sel = mpl.slab_select(sc, cuts, rank)
        ctx.set_stream(stream.cuda_stream)
        mode = "slabs"
    else:
        cuts = None
        ctx = mpl.from_scene(sc, device=local)
        ctx.set_stream(stream.cuda_stream)

    # --restart (default for cfg5B): every step solves the scene's first time step from the same initial
    # state, re-set from a device-resident copy (a D2D copy inside the step), so every step and every GPU
    # count does the same work (strong scaling on a fixed problem; the wheel press hardens as the plate
    # advances: measured 2.8 / 7.8 / 15.8 s for its first three steps on one GPU)
    restart = args.restart if args.restart is not None else sc.name.startswith("cfg5")
    if restart:
        idx = np.arange(sc.n_particles) if sel is None else sel
        dt_ = torch.float32 if args.precision == 32 else torch.float64
        dev0 = [torch.from_numpy(np.ascontiguousarray(a[idx])).to(device="cuda", dtype=dt_)
                for a in (sc.x, sc.v, sc.F, sc.G, sc.vol)]
        mat0 = torch.from_numpy(np.ascontiguousarray(sc.mat[idx])).to("cuda")
        ids0 = None if sel is None else sel.astype(np.int32)

    def one_step():
        if restart:
            ctx.set_particles(*dev0, mat0)
            if ids0 is not None:
                ctx.set_particle_ids(ids0)
        return ctx.step(sc.dt, solver)

    for _ in range(args.warmup):
        one_step()
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    stats = []
    with ClockSampler(local) as clk:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            stats.append(one_step())
        e1.record(stream)
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
    ms_total = e0.elapsed_time(e1)
    n_hvp = sum(s["n_hvp"] for s in stats)
    hvp_ms = sum(s["hvp_ms"] for s in stats)
    cells = statistics.mean(s["n_cells"] for s in stats)
    nodes = statistics.mean(s["n_nodes"] for s in stats)
    # HVP DOF throughput: each step's free DOFs (owned, so a shared node counts once) times its HVPs
    dof_hvp = sum(3.0 * s["n_free_nodes"] * s["n_hvp"] for s in stats)
    n_free = statistics.mean(s["n_free_nodes"] for s in stats)
    ms_per_step = ms_total / args.steps
    launches = float(sum(s["n_launches"] for s in stats))
    if ws > 1:
        # max over ranks of the times; sums of the work (HVP time includes its halo + p.Hp allreduce)
        ms_per_step, hvp_ms_max = pdist.reduce_scalars([ms_per_step, hvp_ms], "max", device="cuda")
        dof_hvp, cells_all, nodes_all, n_free_all, launches = pdist.reduce_scalars(
            [dof_hvp, cells, nodes, n_free, launches], "sum", device="cuda")
    else:
        hvp_ms_max, cells_all, nodes_all, n_free_all = hvp_ms, cells, nodes, n_free
    gdofs = dof_hvp / (hvp_ms_max * 1e-3) / 1e9 if hvp_ms_max > 0 else 0.0
    avg_hvp_ms = hvp_ms_max / max(n_hvp, 1)
    # roofline of the dominant kernel on this rank (rank 0's HVP launches)
    nbytes = hvp_bytes(cells, nodes, 4 if args.precision == 32 else 8)
    fbytes = (cells * KC_REALS * 4 + nodes * 7 * 4) if stats[-1].get("tangent_format") else nbytes
    peak, peak_kind = load_peaks()
    avg_local = hvp_ms / max(n_hvp, 1)
    achieved = nbytes / (avg_local * 1e-3) / 1e9 if avg_local > 0 else 0.0
    # e2e: the same metric through the C ABI with HOST buffers (H2D of particles, D2H of results)
    e2e = None if args.no_e2e else run_e2e(ctx, sc, solver, args, sel, ws)
    clocks = clk.summary()
    vec_ev = os.environ.get("MPL_VEC_EVENTS", "0") in ("1", "2")
    result = {
        "metric": "HVP GDOF/s (matrix-free incremental-potential Hessian-vector product inside Newton-PCG)",
        "value": round(gdofs, 3),
        "unit": "GDOF/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_per_step, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32" if args.precision == 32 else "f64",
        "data": "synthetic (seeded scene generator, paper_2602_07853_b200/scenes.py)",
        "config": {
            "workload": workload_name(sc),
            "grid": list(sc.n), "particles": sc.n_particles, "quadrature_points": int(cells_all),
            "active_nodes": int(nodes_all), "free_dofs": int(3 * n_free_all),
            "parallelism": "1 GPU" if ws == 1 else
            (f"x-slab decomposition over {ws} GPUs (cuts {list(map(int, cuts))} in 4-cell blocks; "
             "halo sums + allreduces on the library's NCCL communicator)"),
            "l2": "inputs larger than L2 (tangent stream > 126 MB per HVP)",
            "step": "full implicit step: resample + Newton-PCG + G2P" + (
                " (each step restarts from the initial state: fixed work per step)" if restart else " (consecutive steps)"),
            "solver": {"eps_cg": solver.eps_cg, "eps_newton": solver.eps_newton, "psd": bool(getattr(solver, "psd", False)),
                       "newton_max": solver.newton_max, "cg_max": solver.cg_max,
                       "pcg": os.environ.get("MPL_PCG", "cg1" if ws > 1 else "classic")},
        },
        "implicit_step_ms": round(ms_per_step, 3),
        "newton_iters": [s["newton_iters"] for s in stats],
        "cg_iters": [s["cg_iters"] for s in stats],
        "hvp_ms": round(avg_hvp_ms, 5),
        "hvp_per_s": round(1e3 / avg_hvp_ms, 1) if avg_hvp_ms > 0 else None,
        "qp_per_s": round(cells_all / (avg_hvp_ms * 1e-3), 1) if avg_hvp_ms > 0 else None,
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": load_traffic(sc.name, hvp_kernel_name(args.precision)) if ws == 1 and stats[-1].get("tangent_format") else None,
                     "peak_kind": peak_kind, "kernel": hvp_kernel_name(args.precision),
                     "tangent": f"compressed ({KC_REALS} reals per quadrature point)" if stats[-1].get("tangent_format") else
                                "45 reals per quadrature point",
                     "algorithmic_bytes_per_launch": int(nbytes), "pct_of_8TBps": round(achieved / 8000.0, 4),
                     # the bytes the compressed format itself must move (96 B per quadrature point + 28 B per
                     # node), and the fraction of peak on that count: the metric keeps SURVEY §8(d)'s figure
                     "format_bytes_per_launch": int(fbytes),
                     "format_frac": round(fbytes / (avg_local * 1e-3) / 1e9 / peak, 4) if avg_local > 0 else None},
        "e2e": e2e,
        "gpu_launches": int(launches),
        "converged": [bool(s["converged"]) for s in stats],
        "all_converged": all(bool(s["converged"]) for s in stats),
        "grad_rel": [s["grad_norm"] / s["grad_norm0"] if s["grad_norm0"] > 0 else 0.0 for s in stats],
        "ls_halvings": [s["ls_halvings"] for s in stats],
        "phase_ms": {"resample": round(statistics.mean(s["ms_phase"][0] for s in stats), 3),
                     "linearize": round(statistics.mean(s["ms_phase"][3] for s in stats), 3),
                     "pcg": round(statistics.mean(s["ms_phase"][4] for s in stats), 3),
                     # measured only with MPL_VEC_EVENTS=1 (events around every vector kernel)
                     "pcg_vector_kernels": round(statistics.mean(s["ms_phase"][1] for s in stats), 3) if vec_ev else None,
                     "pcg_update2": round(statistics.mean(s["ms_phase"][2] for s in stats), 3) if vec_ev else None,
                     "line_search": round(statistics.mean(s["ms_phase"][5] for s in stats), 3),
                     "g2p": round(statistics.mean(s["ms_phase"][6] for s in stats), 3)},
        "clocks": clocks,
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        result["cpu_baseline"] = cpu_baseline(sc, args)
    if not result["all_converged"]:
        # a step that hit newton_max is not a converged implicit step: say so in the line and on stderr
        result["invalid"] = "a timed step did not converge (newton_max reached); see grad_rel"
        if rank == 0:
            print("bench: WARNING: " + result["invalid"], file=sys.stderr, flush=True)
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()
    if ws > 1:
        dist.destroy_process_group()


def run_e2e(ctx, sc, solver, args, sel, ws):
    """Same metric through the C ABI with host buffers: each step copies the (rank's) particle state
    from pinned host memory (H2D), steps, and reads the particle state back (D2H).  On one GPU the
    copies are pipelined with the solve (mpl_stage_particles / mpl_get_particles_async on the
    library's two copy streams); slab ranks copy synchronously.  Wall clock, max over ranks."""
    import torch
    dt_ = torch.float32 if args.precision == 32 else torch.float64
    idx = np.arange(sc.n_particles) if sel is None else sel
    host = [torch.from_numpy(np.ascontiguousarray(a[idx])).to(dt_).pin_memory() for a in (sc.x, sc.v, sc.F, sc.G, sc.vol)]
    mat = torch.from_numpy(np.ascontiguousarray(sc.mat[idx])).pin_memory()
    cap = int(len(idx) * 1.25) + 1024
    outs = [torch.empty((cap, w), dtype=dt_).pin_memory() for w in (3, 3, 9, 9)]
    s = 4 if args.precision == 32 else 8
    n = len(idx)
    h2d = n * (3 + 3 + 9 + 9 + 1) * s + n * 4
    steps = 20  # the pipeline fills (first upload) and drains (last readback) once per measurement
    n_hvp_dofs = 0.0
    d2h = 0
    single = sel is None  # one GPU, or a full-scene replica per rank: the pipelined single-context path
    if single:  # untimed warm-up of the pipelined path (staging / readback buffers, copy streams)
        ctx.stage_particles(*host, mat)
        ctx.resample(sc.dt)
        ctx.newton_step(solver)
        ctx.transfer_to_particles(sc.dt)
        ctx.get_particles_async(*[o[:n] for o in outs])
        ctx.stage_wait()
    torch.cuda.synchronize()
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
    t0 = time.perf_counter()
    if single:
        # pipelined through the public API: step s+1's inputs go up (H2D copy stream) while step s
        # solves, step s's result comes down (D2H copy stream) while step s+1 runs
        ctx.stage_particles(*host, mat)
        for i in range(steps):
            ctx.resample(sc.dt)  # adopts the staged inputs of this step
            if i + 1 < steps:
                ctx.stage_particles(*host, mat)
            st = ctx.newton_step(solver)
            ctx.transfer_to_particles(sc.dt)
            k = ctx.num_particles()
            ctx.get_particles_async(*[o[:k] for o in outs])
            d2h = k * (3 + 3 + 9 + 9) * s
            n_hvp_dofs += 3.0 * st["n_free_nodes"] * st["n_hvp"]
        ctx.stage_wait()
    else:
        for _ in range(steps):
            ctx.set_particles(*host, mat)
            ctx.set_particle_ids(sel.astype(np.int32))
            st = ctx.step(sc.dt, solver)
            k = ctx.num_particles()
            ctx.get_particles(*[o[:k] for o in outs])
            d2h = k * (3 + 3 + 9 + 9) * s
            n_hvp_dofs += 3.0 * st["n_free_nodes"] * st["n_hvp"]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if ws > 1:
        from paper_2602_07853_b200 import dist as pdist
        wall, = pdist.reduce_scalars([wall], "max", device="cuda")
        n_hvp_dofs, h2d, d2h = pdist.reduce_scalars([n_hvp_dofs, h2d, d2h], "sum", device="cuda")
    val = n_hvp_dofs / wall / 1e9
    return {"value": round(val, 3), "unit": "GDOF/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "ms_per_step": round(wall * 1e3 / steps, 3), "steps": steps,
            "mode": ("pipelined: every step uploads the same host particle state (independent steps), so step s+1's "
                     "upload overlaps step s's solve and step s's readback overlaps step s+1" if single else
                     "synchronous per step on slab ranks (set_particles, step, get_particles)")}


# ------------------------------------------------------------------------------------------------
def oracle_window(sc, lo, size):
    """A window of the scene (cells [lo, lo+size)^3) for the oracle: particles whose stencil can touch
    it, grid origin shifted; interior outputs equal the full-scene values."""
    import oracle
    from paper_2602_07853_b200 import scenes
    lo = np.asarray(lo)
    x = sc.x.astype(np.float64)
    cell = np.floor(x / sc.dx - 0.5).astype(np.int64)
    keep = np.all((cell >= lo - 1) & (cell <= lo + size), axis=1)
    sub = scenes.subset(sc, keep)
    grid = oracle.Grid((size + 2,) * 3, sc.dx, tuple((lo - 1) * sc.dx))
    un, S, prob, v0 = oracle.prepare(sub, grid, clip=True)
    return grid, un, S, prob, v0


def _omp_threads(n: int) -> None:
    """Thread count of the oracle's OpenMP colour loops (libgomp is loaded with liboracle.so)."""
    import ctypes
    try:
        ctypes.CDLL("libgomp.so.1").omp_set_num_threads(int(n))
    except OSError:
        pass


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(sc, args, budget_s=10.0):
    """Oracle HVP (plain fp64 C; OpenMP colour loops, identical results at any thread count) on a bounded
    window of the same workload, on all host cores and on one core (SURVEY §8(d) timing protocol)."""
    import oracle
    lo, size = _window_for(sc)
    grid, un, S, prob, v0 = oracle_window(sc, lo, size)
    rng = np.random.default_rng(4)
    act = (prob.m_i > 0)
    u = rng.normal(size=v0.shape) * act[:, None]
    n_free = int(prob.freed.sum())
    ncores = os.cpu_count() or 1
    out = {}
    for cores in (ncores, 1):
        _omp_threads(cores)
        prob.hvp(v0, u)  # warm-up
        t0 = time.perf_counter()
        reps = 0
        while True:
            prob.hvp(v0, u)
            reps += 1
            if time.perf_counter() - t0 > budget_s:
                break
        out[cores] = ((time.perf_counter() - t0) / reps, reps)
    _omp_threads(ncores)
    t, reps = out[ncores]
    t1, reps1 = out[1]
    sample = (f"oracle HVPs on the {size}^3-cell window at cells {list(map(int, lo))} of {sc.name} "
              f"({int((un.m_c > 0).sum())} quadrature points, {n_free} free nodes): {reps} runs on {ncores} threads, "
              f"{t * 1e3:.2f} ms each; {reps1} runs on 1 thread, {t1 * 1e3:.2f} ms each")
    return {"value": round(3.0 * n_free / t / 1e9, 6), "unit": "GDOF/s", "cores": ncores, "kind": "oracle",
            "sample": sample, "cpu_model": _cpu_model(), "nproc": ncores,
            "single_core": {"value": round(3.0 * n_free / t1 / 1e9, 6), "cores": 1}}


def _window_for(sc):
    n = sc.n[0]
    if sc.name.startswith("cfg4"):
        return np.array([int(0.25 * n) - 12, int(0.35 * n) - 12, int(0.5 * n) - 12]), 24
    if sc.name.startswith("cfg5"):
        return np.array([int(0.5 * n) - 12, int(0.1 * n), int(0.5 * n) - 12]), 24
    c = n // 2
    return np.array([c - 12] * 3), 24


def run_reference(args):
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from paper_2602_07853_b200 import scenes
    sc = scenes.by_name(args.config, args.precision)
    import oracle
    lo, size = _window_for(sc)
    grid, un, S, prob, v0 = oracle_window(sc, lo, size)
    rng = np.random.default_rng(4)
    u = rng.normal(size=v0.shape) * (prob.m_i > 0)[:, None]
    n_free = int(prob.freed.sum())
    ncores = os.cpu_count() or 1
    _omp_threads(ncores)
    for _ in range(args.warmup):
        prob.hvp(v0, u)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        prob.hvp(v0, u)
    t = (time.perf_counter() - t0) / args.steps
    val = 3.0 * n_free / t / 1e9
    sample = (f"one oracle HVP per step on the {size}^3-cell window at cells {list(map(int, lo))} of {sc.name} "
              f"({n_free} free nodes), {ncores} OpenMP threads")
    print(json.dumps({
        "impl": "reference",
        "metric": "HVP GDOF/s (matrix-free incremental-potential Hessian-vector product inside Newton-PCG)",
        "value": round(val, 6), "unit": "GDOF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (same seeded scene, windowed)",
        "config": {"workload": workload_name(sc), "sample": sample, "grid": list(sc.n),
                   "particles": sc.n_particles},
        "cpu_baseline": {"value": round(val, 6), "unit": "GDOF/s", "cores": ncores, "kind": "oracle", "sample": sample,
                         "cpu_model": _cpu_model()},
        "e2e": {"value": round(val, 6), "unit": "GDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None,
                    help="default: cfg4 on one GPU (the 256^3 headline), cfg5B (the 512^3 scaling config) for N > 1")
    ap.add_argument("--precision", type=int, default=32)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--restart", type=int, default=None,
                    help="1: every step restarts from the initial state (default for cfg5B), 0: consecutive steps")
    args = ap.parse_args()
    if args.config is None:
        args.config = "cfg4" if int(os.environ.get("WORLD_SIZE", "1")) <= 1 else "cfg5B"
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
