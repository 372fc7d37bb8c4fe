#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: "BP3 diffusion GDOF/s per GPU
vs p; CG [DOFs x iters]/s at 1/2/4/8 B200").

One *step* = one CG iteration of the BP3 diffusion operator (SURVEY.md §8(a)
rows a4-a10: fused apply + p.Ap + fused updates), p = 5, Gauss Q = p+2,
curvilinear unit cube, homogeneous Dirichlet, manufactured RHS, on BASELINE
config 5's slab of 200 x 200 x 25 elements per GPU (125.5M dofs per GPU; weak
scaling stacks one slab per GPU in z, exchanged over NCCL).  ``value`` = global
DOFs x iterations / s over all GPUs (G[DOF*it]/s), device-timed with CUDA
events, max over ranks.  The line also carries the dominant kernel's roofline
(its launch durations recorded by the library's CUDA events on the launching
stream inside the timed CG region),
e2e (host buffers through the public API), the CPU oracle baseline and -- on
rank 0 at N = 1, time-bounded -- ``sweep``: apply GDOF/s and HBM-roofline
fraction vs p for configs 2-4 (BP3 fused / unfused / fully matrix-free, BP5,
BP1 eager / CUDA-graph / L2-flushed + 100-iteration CG), the DG mass operator,
the DOFs needed to reach 80 % of peak, BPS3 p-multigrid PCG vs CG, and
BASELINE config 4 (BP5 CG to 1e-10, p = 4..8).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--p 5] [--no-sweep] [--no-bp5-cg]
    python bench.py --impl reference ...   # the CPU oracle (rank 0 only)

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BP3 diffusion GDOF/s per GPU vs p; CG [DOFs\u00d7iters]/s at 1/2/4/8 B200"  # BASELINE.json
UNIT = "GDOF*it/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def alg_bytes(nx, ny, nz, p, Q, nc):
    """8 N_L (read x) + 8 N_L (write y) + 8 n_c E Q^3 (qdata)."""
    N = (p * nx + 1) * (p * ny + 1) * (p * nz + 1)
    E = nx * ny * nz
    return 16 * N + 8 * nc * E * Q ** 3, N, E


KERNEL_NAMES = {1: "fused_elem_simt"}  # fused_info.variant


class ClockSampler:
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    def __init__(self, device: int, period=0.02):
        self.device, self.period = device, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            names = {
                "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
                "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
                "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
                "display_clock_setting": 0x100}

            def run():
                while not self._stop.is_set():
                    try:
                        self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                        r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                        for k, v in names.items():
                            if r & v and k != "gpu_idle":
                                self.reasons.add(k)
                    except Exception:
                        pass
                    time.sleep(self.period)
            self._t = threading.Thread(target=run, daemon=True)
            self._t.start()
        except Exception:
            self._t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def cpu_info():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ----------------------------------------------------------------------------- reference arm
def oracle_cg_sample(p, n, iters, warmup=0):
    """The CPU oracle (brute-force EA operator + textbook CG) on a bounded sample
    of the BP3 workload.  Returns (dofs*iters/s, setup_s, cg_s, dofs, threads)."""
    import oracle as O
    om = O.Mesh(n, n, n, p, alpha=0.1)
    t0 = time.perf_counter()
    Ae = O.element_matrices(om, O.DIFFUSION, O.GAUSS)
    b = O.rhs(om, O.DIFFUSION, O.GAUSS, bc=1)
    t1 = time.perf_counter()
    if warmup:
        O.cg(b, m=om, Ae=Ae, bc=1, max_iter=warmup, fixed_iters=True)
    t2 = time.perf_counter()
    O.cg(b, m=om, Ae=Ae, bc=1, max_iter=iters, fixed_iters=True)
    t3 = time.perf_counter()
    return om.n_dofs * iters / (t3 - t2), t1 - t0, t3 - t2, om.n_dofs, O.num_threads()


def slab_dims(args):
    """Per-GPU slab (elements): BASELINE config 5: 200 x 200 x 25
    per GPU, stacked in z for weak scaling; --n gives an n^3 slab instead."""
    if args.n:
        return args.n, args.n, args.n
    return tuple(int(v) for v in args.slab.split(","))


def arm_config(p, dims, world):
    """The workload both arms report."""
    nx, ny, nzs = dims
    Q = p + 2
    n_global = (p * nx + 1) * (p * ny + 1) * (p * nzs * world + 1)
    qd_gb = nx * ny * nzs * 6 * Q ** 3 * 8 / 1e9
    vec_mb = (p * nx + 1) * (p * ny + 1) * (p * nzs + 1) * 8 / 1e6
    return {"workload": f"bp3_p{p}_{nx}x{ny}x{nzs}_per_gpu (BASELINE config 5, weak scaling)",
            "p": p, "q": Q, "elements_per_gpu": nx * ny * nzs, "dofs_global": n_global,
            "dofs_per_gpu_local": (p * nx + 1) * (p * ny + 1) * (p * nzs + 1), "bc": "dirichlet",
            "mesh": "curvilinear alpha=0.1",
            "parallelism": f"z-slab x{world} (NCCL plane exchange + allreduce)",
            "l2": f"inputs larger than L2 (qdata {qd_gb:.1f} GB/GPU, vectors {vec_mb:.0f} MB), no flush"}


def run_oracle_plan(args):
    """SURVEY.md §8(d) oracle timing plan, on the host cores: EA setup (the
    "Element Assembly" level), EA apply and 10 fixed CG
    iterations timed separately (median of 3), with 1 thread and all cores, on
    the per-config sample sizes; prints one JSON line (rank 0 only)."""
    import oracle as O
    import workloads as W
    if int(os.environ.get("RANK", "0")) != 0:
        return
    ncores = os.cpu_count() or 1
    plan = [("config1_bp3_2x2x2_p2", O.DIFFUSION, O.GAUSS, 2, (2, 2, 2), 1)]
    plan += [(f"config2_bp1_p{p}", O.MASS, O.GAUSS, p, (W.bp1_sweep_n(p),) * 3, 0)
             for p in (1, 2, 3, 4, 5)]
    plan += [(f"config3_bp3_p{p}_n_over_4", O.DIFFUSION, O.GAUSS, p,
              (max(1, W.bp3_sweep_n(p) // 4),) * 3, 1) for p in (2, 5)]
    plan += [("config4_bp5_p5_n8", O.DIFFUSION, O.GLL, 5, (8, 8, 8), 1),
             ("config5_bp3_p5_16x16x2", O.DIFFUSION, O.GAUSS, 5, (16, 16, 2), 1)]
    rows = []
    for name, kind, rule, p, dims, bc in plan:
        om = O.Mesh(*dims, p, alpha=0.1)
        x = W.random_vector(1, np.arange(om.n_dofs))
        b = O.rhs(om, kind, rule, bc=bc)
        row = {"case": name, "p": p, "elements": dims, "dofs": om.n_dofs}
        for threads in sorted({1, ncores}):
            O.set_threads(threads)
            ts, ta, tc = [], [], []
            for _ in range(3):
                t0 = time.perf_counter()
                Ae = O.element_matrices(om, kind, rule)
                t1 = time.perf_counter()
                O.apply_ea(om, Ae, x, bc=bc)
                t2 = time.perf_counter()
                O.cg(b, m=om, Ae=Ae, bc=bc, max_iter=10, fixed_iters=True)
                t3 = time.perf_counter()
                ts.append(t1 - t0); ta.append(t2 - t1); tc.append(t3 - t2)
                del Ae
            sa, aa, ca = (statistics.median(v) for v in (ts, ta, tc))
            row[f"threads_{threads}"] = {"setup_s": sa, "apply_s": aa, "cg10_s": ca,
                                         "apply_gdof_s": om.n_dofs / aa / 1e9,
                                         "cg_gdof_it_s": om.n_dofs * 10 / ca / 1e9}
        rows.append(row)
    O.set_threads(ncores)
    print(json.dumps({"oracle_plan": rows, "cpu": cpu_info(), "cores": ncores}), flush=True)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p, n = args.p, args.ref_n
    val, setup_s, cg_s, dofs, threads = oracle_cg_sample(p, n, args.steps, args.warmup)
    v = val / 1e9
    sample = (f"BP3 p={p} on {n}^3 elements ({dofs} dofs), brute-force EA setup {setup_s:.1f} s "
              f"(untimed), {args.steps} timed fixed CG iterations ({cg_s:.2f} s); CPU {cpu_info()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * cg_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        # the arm's workload; each step is the bounded oracle sample named in cpu_baseline
        "config": arm_config(p, slab_dims(args), args.gpus),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2402_15940_b200 as hf

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    comm = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        comm = hf.Comm.from_torch_distributed()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    p = args.p
    nx, ny, nzs = slab_dims(args)
    nz = nzs * world
    Q = p + 2
    mesh = hf.Mesh(nx, ny, nz, p, alpha=0.1, comm=comm)
    op = hf.Operator(mesh, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    b = op.rhs()
    x = torch.zeros(mesh.n_local, dtype=torch.float64, device=dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up: W CG iterations
    op.cg(b, x, max_iter=max(args.warmup, 1), fixed_iters=True)

    # ---- timed: exactly K CG iterations (one hofem_cg call in fixed-iteration mode;
    # its initial residual apply is inside the timed region and not counted)
    x.zero_()
    barrier()
    hf.launch_count_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the dominant kernel's launch durations are recorded live inside the timed
    # region: CUDA events the library puts around each brick launch on its stream
    # (hofem_profile_*; two event records per launch, no synchronization)
    hf.profile_enable(True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        st, stats, _ = op.cg(b, x, max_iter=args.steps, fixed_iters=True)
        e1.record(stream)
        barrier()
    prof = hf.profile_read()
    hf.profile_enable(False)
    launches = hf.launch_count()
    t_cg = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    assert stats.iterations == args.steps
    n_global = mesh.n_global
    value = n_global * args.steps / t_cg / 1e9

    # ---- apply-only: GDOF/s per GPU + live per-kernel durations (profiling hooks)
    xa = mesh.random(1)
    ya = torch.empty_like(xa)
    for _ in range(3):
        op.apply(xa, ya)
    napply = args.apply_reps
    barrier()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record(stream)
    for _ in range(napply):
        op.apply(xa, ya)
    a1.record(stream)
    barrier()
    t_apply = max_over_ranks(a0.elapsed_time(a1) / 1e3 / napply)
    t_brick = max_over_ranks(prof.brick_ms / 1e3 / max(prof.brick_launches, 1))
    t_fix = prof.fixup_ms / 1e3 / max(prof.fixup_launches, 1)
    bytes_apply, N_l, E_l = alg_bytes(nx, ny, nzs, p, Q, 6)
    info = op.fused_info()
    nd = info.direct_points
    bytes_brick = 8 * N_l + 8 * 6 * E_l * Q ** 3 + 8 * nd
    peak, peak_src = load_peaks()
    achieved = bytes_brick / t_brick / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            ent = json.load(open(tpath)).get(f"bp3_p{p}_{nx}x{ny}x{nzs}")
            traffic = ent["dram_bytes"] if ent else None
        except Exception:
            traffic = None

    # ---- e2e: public API with host buffers (H2D b, solve, D2H x) per solve
    e2e = None
    if not args.no_e2e:
        hb = torch.empty(mesh.n_local, dtype=torch.float64, pin_memory=True)
        hb.copy_(b.cpu())
        hx = torch.empty(mesh.n_local, dtype=torch.float64, pin_memory=True)
        db = torch.empty_like(b)
        it = args.e2e_iters
        reps = args.e2e_reps
        barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(reps):
            db.copy_(hb, non_blocking=True)
            x.zero_()
            op.cg(db, x, max_iter=it, fixed_iters=True)
            hx.copy_(x, non_blocking=True)
        s1.record(stream)
        barrier()
        t_e2e = max_over_ranks(s0.elapsed_time(s1) / 1e3)
        e2e = {"value": n_global * it * reps / t_e2e / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 8 * mesh.n_local, "d2h_bytes_per_step": 8 * mesh.n_local,
               "step": f"one hofem_cg solve of {it} fixed iterations incl. H2D of b and D2H of x "
                       f"(per rank); {reps} solves timed"}

    # ---- sweep (rank 0, N = 1; time-bounded): configs 2-4 and the §8(f) rows
    sweep = None
    if rank == 0 and world == 1 and not args.no_sweep:
        op.close()
        mesh.close()
        del b, x
        torch.cuda.empty_cache()
        sweep = run_sweep(args, hf, torch, stream)

    # ---- CPU baseline: rank 0, N = 1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, setup_s, cg_s, dofs, threads = oracle_cg_sample(p, args.ref_n, args.ref_iters)
        cpu = {"value": v / 1e9, "unit": UNIT, "cores": threads, "kind": "oracle",
               "sample": f"BP3 p={p} on {args.ref_n}^3 elements ({dofs} dofs): brute-force EA "
                         f"setup {setup_s:.1f} s (excluded), {args.ref_iters} fixed CG iterations "
                         f"in {cg_s:.2f} s; CPU {cpu_info()}"}

    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_cg / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": arm_config(p, (nx, ny, nzs), world),
            "apply_gdof_s_per_gpu": N_l / t_apply / 1e9,
            "apply_ms": 1e3 * t_apply,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": f"{KERNEL_NAMES.get(info.variant, '?')}<DIFF,P1={p + 1},Q={Q}>"
                                   f" brick {info.bx}x{info.by}x1, {info.grid} CTAs",
                         "alg_bytes_per_launch": bytes_brick, "launch_ms": 1e3 * t_brick,
                         "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_src})",
                         "apply_frac": bytes_apply / t_apply / 1e9 / peak,
                         "fixup_ms": 1e3 * t_fix,
                         "launches_timed": prof.brick_launches,
                         "timed_in": "the timed CG region (library CUDA events around each "
                                     "brick launch on its stream)"},
            "gpu_launches": launches,
            "clocks": clocks,
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if sweep is not None:
            line["sweep"] = sweep
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _evt_time(torch, stream, fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def _graph_time(torch, fn, reps=200, launches=5):
    """`reps` applies captured in ONE CUDA graph, median
    of `launches` graph launches (per apply)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    ts = []
    for _ in range(launches):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / reps)
    del g
    return statistics.median(ts)


def run_sweep(args, hf, torch, stream):
    """Configs 2-4 of BASELINE.json and the §8(f) rows, time-bounded: apply
    throughput per GPU vs p with its HBM-roofline fraction (algorithmic bytes,
    SURVEY.md §8(d)), fused / unfused / fully matrix-free BP3, BP5, BP1 (eager,
    CUDA-graph, L2-flushed; 100-iteration CG), DG mass; the DOFs needed to reach
    80 % of peak; BPS3 p-multigrid PCG vs CG."""
    import workloads as W
    peak, _ = load_peaks()
    out = {"bp3": [], "bp5": [], "bp1": [], "dg": []}
    reps = args.sweep_reps

    def rec(name, t, nbytes, ndofs, flops=None):
        d = {"ms": 1e3 * t, "gdof_s": ndofs / t / 1e9, "alg_gbs": nbytes / t / 1e9,
             "frac": nbytes / t / 1e9 / peak}
        if flops:
            d["fp64_tflops"] = flops / t / 1e12
        return d

    for bench, kind, rule, ps in (("bp3", hf.DIFFUSION, hf.GAUSS, range(1, 9)),
                                  ("bp5", hf.DIFFUSION, hf.GLL, range(4, 9)),
                                  ("bp1", hf.MASS, hf.GAUSS, range(1, 9))):
        for p in ps:
            n = W.bp1_sweep_n(p) if bench == "bp1" else W.bp3_sweep_n(p)
            Q = p + 2 if rule == hf.GAUSS else p + 1
            nc = 1 if kind == hf.MASS else 6
            m = hf.Mesh(n, n, n, p, alpha=0.1)
            op = hf.Operator(m, kind=kind, rule=rule)
            x = m.random(3)
            y = torch.empty_like(x)
            bts, N, E = alg_bytes(n, n, n, p, Q, nc)
            res = {"p": p, "n": n, "dofs": N}
            res["fused"] = rec("fused", _evt_time(torch, stream, lambda: op.apply(x, y), reps),
                               bts, N)
            if bench == "bp3":
                res["unfused"] = rec("unfused", _evt_time(torch, stream,
                                                          lambda: op.apply_unfused(x, y),
                                                          max(3, reps // 4)), bts, N)
                # f3: algorithmic bytes 8 (x) + 24 (X, Y, Z) + 8 (y) B/DOF + the
                # E-vector round trip 16 B per element dof
                bmf = 40 * N + 16 * E * (p + 1) ** 3
                res["matrix_free"] = rec("mf", _evt_time(torch, stream,
                                                         lambda: op.apply_mf(x, y),
                                                         max(3, reps // 4)), bmf, N)
            if bench == "bp1":
                res["graph"] = rec("graph", _graph_time(torch, lambda: op.apply(x, y),
                                                       reps=200), bts, N)
                # cold L2: a 2 x L2 memset between applies; its own time subtracted
                flush = torch.empty(2 * 126 * 2 ** 20 // 8, dtype=torch.float64, device="cuda")
                t_fl = _evt_time(torch, stream, lambda: flush.zero_(), 10)
                t_both = _evt_time(torch, stream, lambda: (flush.zero_(), op.apply(x, y)), 10)
                res["l2_flushed"] = rec("flushed", max(t_both - t_fl, 1e-9), bts, N)
                del flush
                b = op.rhs()
                xs = torch.zeros_like(b)
                t_cg = _evt_time(torch, stream,
                                 lambda: op.cg(b, xs, max_iter=100, fixed_iters=True), 1, warm=1)
                res["cg_100"] = {"ms": 1e3 * t_cg, "gdof_it_s": N * 100 / t_cg / 1e9,
                                 "us_per_it": 1e4 * t_cg}
            out[bench].append(res)
            op.close()
            m.close()
            torch.cuda.empty_cache()
    # f4: DG (L2) mass, ~30M DG dofs
    for p in range(1, 9):
        n = W.dg_sweep_n(p)
        m = hf.Mesh(n, n, n, p, alpha=0.1)
        dg = hf.DGMass(m)
        x = dg.random(1)
        y = torch.empty_like(x)
        E = n ** 3
        bts = 16 * dg.n_local + 8 * E * (p + 2) ** 3
        r = rec("dg", _evt_time(torch, stream, lambda: dg.apply(x, y), reps), bts, dg.n_local)
        r.update({"p": p, "n": n, "dofs": dg.n_local})
        out["dg"].append(r)
        dg.close()
        m.close()
        torch.cuda.empty_cache()
    # f1 metric: DOFs needed to reach 80 % of peak, BP3 p=5 CG
    # iterations, fused schedule (in-kernel fix-up + fused update / persistent
    # kernel, i.e. the defaults) vs the separate-kernel schedule
    sizes = [4, 6, 8, 12, 16, 20, 24, 28, 32, 38, 44, 52, 62]
    curves = {"fused": [], "separate": []}
    for n in sizes:
        m = hf.Mesh(n, n, n, 5, alpha=0.1)
        op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
        b = op.rhs()
        xs = torch.zeros_like(b)
        for name in ("fused", "separate"):
            v = hf.AUTO if name == "fused" else hf.NEVER
            for o in (hf.OPT_INFIX, hf.OPT_CG_FUSED_UPDATE, hf.OPT_CG_PERSISTENT):
                op.set_option(o, v)
            it = 50
            t = _evt_time(torch, stream, lambda: op.cg(b, xs, max_iter=it, fixed_iters=True), 1,
                          warm=1)
            curves[name].append({"n": n, "dofs": m.n_local, "gdof_it_s": m.n_local * it / t / 1e9})
        op.close()
        m.close()
        torch.cuda.empty_cache()
    d80, d80i = {}, {}
    for name, cv in curves.items():
        top = max(c["gdof_it_s"] for c in cv)
        k = next(i for i, c in enumerate(cv) if c["gdof_it_s"] >= 0.8 * top)
        d80[name] = cv[k]["dofs"]
        d80i[name] = cv[k]["dofs"]
        if k > 0:  # crossing, interpolated linearly in log(dofs)
            a, b = cv[k - 1], cv[k]
            f = (0.8 * top - a["gdof_it_s"]) / (b["gdof_it_s"] - a["gdof_it_s"])
            d80i[name] = int(round(np.exp(np.log(a["dofs"]) +
                                          f * (np.log(b["dofs"]) - np.log(a["dofs"])))))
    out["dofs_to_80pct_of_peak"] = {"bench": "bp3 p=5 CG (Dirichlet), 50 fixed iterations",
                                    "curves": curves, "dofs_80pct": d80,
                                    "dofs_80pct_interpolated": d80i,
                                    "peak": {k: max(c["gdof_it_s"] for c in v)
                                             for k, v in curves.items()}}
    # f2: BPS3 -- p-multigrid preconditioned CG vs CG to 1e-10 (BP3 p=5, 24^3 elements)
    m = hf.Mesh(24, 24, 24, 5, alpha=0.1)
    op = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GAUSS, bc=hf.BC_DIRICHLET)
    b = op.rhs()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    P = hf.PMG(m, degree=3)
    t_setup = time.perf_counter() - t0
    xs = torch.zeros_like(b)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, pst, _ = P.pcg(b, xs, rel_tol=1e-10, max_iter=500)
    t_pcg = time.perf_counter() - t0
    xs.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    _, cst, _ = op.cg(b, xs, rel_tol=1e-10, max_iter=20000, check_every=10)
    t_cgs = time.perf_counter() - t0
    out["bps3"] = {"mesh": "24^3 elements, p=5, curvilinear, Dirichlet", "dofs": m.n_local,
                   "orders": P.orders, "chebyshev_degree": 3,
                   "pmg_pcg": {"iterations": pst.iterations, "s": t_pcg, "setup_s": t_setup,
                               "rel_res": pst.final_rel_res},
                   "cg": {"iterations": cst.iterations, "s": t_cgs, "rel_res": cst.final_rel_res}}
    P.close()
    op.close()
    m.close()
    torch.cuda.empty_cache()
    if not getattr(args, "no_bp5_cg", False):
        out["bp5_cg_1e-10"] = []
        for p in range(4, 9):
            n = W.bp3_sweep_n(p)
            m = hf.Mesh(n, n, n, p, alpha=0.1)
            opd = hf.Operator(m, kind=hf.DIFFUSION, rule=hf.GLL, bc=hf.BC_DIRICHLET)
            b = opd.rhs()
            xs = torch.zeros_like(b)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            st, stats, _ = opd.cg(b, xs, rel_tol=1e-10, max_iter=20000, check_every=50)
            t = time.perf_counter() - t0
            out["bp5_cg_1e-10"].append({"p": p, "iterations": stats.iterations, "s": t,
                                        "gdof_it_s": m.n_local * stats.iterations / t / 1e9})
            opd.close()
            m.close()
            torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--p", type=int, default=5)
    ap.add_argument("--n", type=int, default=0, help="n^3 elements per GPU instead of --slab")
    ap.add_argument("--slab", default="200,200,25",
                    help="elements per GPU nx,ny,nz (BASELINE config 5: 200,200,25)")
    ap.add_argument("--apply-reps", type=int, default=50)
    ap.add_argument("--e2e-iters", type=int, default=100)
    ap.add_argument("--e2e-reps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--ref-n", type=int, default=10, help="oracle sample: elements per axis")
    ap.add_argument("--ref-iters", type=int, default=3000)
    ap.add_argument("--no-sweep", action="store_true", help="skip the p / size sweeps")
    ap.add_argument("--oracle-plan", action="store_true",
                    help="SURVEY §8(d) oracle timing plan on the host cores (no GPU work)")
    ap.add_argument("--sweep-reps", type=int, default=20)
    ap.add_argument("--no-bp5-cg", action="store_true",
                    help="skip the sweep's BP5 CG solves to 1e-10 (BASELINE config 4, ~15 s)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.oracle_plan:
        run_oracle_plan(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
