"""Benchmark: CG GDOF/s (N=7, FP64) and time per CG iteration.

Workload (BASELINE.json configs[2]/[3]): Poisson PCG
(h1=1, h2=0, Jacobi on the assembled diagonal, multiplicity-weighted dots) on
the 64^3-element deformed unit box (a = 0.05), N = 7 -- 262,144 elements,
134,217,728 local nodes -- solved from a zero initial guess.  One "step" is
one PCG solve run for a fixed ITERS iterations (tolerance 0, so every step
does identical work).  GDOF/s counts local nodes, E*(N+1)^3 * iterations /
seconds (proj/src/bench.cpp:168).  Multi-GPU: the same mesh partitioned by
RCB across the ranks (strong scaling).

Arms:
  default            our CUDA path (libsbx.so).  `value`: device-resident
                     b/x, CUDA-event timed; `e2e`: the C-ABI call with pinned
                     HOST b/x (H2D of b and x0, D2H of x inside the timing).
  --impl reference   the reference's own CPU pcg (oracle/_ref, compiled from
                     /root/reference, all host threads) on a bounded sample.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG GDOF/s (N=7, FP64, Poisson PCG+Jacobi, deformed box)"
UNIT = "GDOF/s"


def unique_fraction(ex, ey, ez, N):
    """unique / local DOF of a non-periodic box (SURVEY §8(d) DOF convention)."""
    return (ex * N + 1) * (ey * N + 1) * (ez * N + 1) / (ex * ey * ez * (N + 1) ** 3)


def k1_geometry(N):
    """Which K1 variant the fused CG runs (mirrors launch_k1 in cg.cu): box
    contexts with an even node count 8 <= n = N+1 <= 16, and n = 6 on the
    tensor cores, form the metric on the fly from the trilinear map (56 B/node
    + 192 B/element streamed); otherwise the 6 stored factors are streamed
    (104 B/node)."""
    n = N + 1
    if (os.environ.get("SBX_STORED_GEOMETRY") or os.environ.get("SBX_NO_TMA") or n % 2
            or n > 16 or n < 6):
        return "stored"
    if n == 6 and (os.environ.get("SBX_K1_FMA") or os.environ.get("SBX_K1_FMAG")):
        return "stored"
    return "trilinear"


def roofline_block(N, E, nodes, k1_ms, k2_ms, it_ms, peak, peak_kind, traffic, kernel):
    """Roofline of the dominant kernel (K1) plus the whole iteration, from
    ALGORITHMIC bytes."""
    geo = k1_geometry(N)
    k1_bytes = (7 * 8 * nodes + 24 * 8 * E) if geo == "trilinear" else 13 * 8 * nodes
    it_bytes = k1_bytes + 4 * 8 * nodes  # + K2: w, r, 1/diag read, r written
    achieved = k1_bytes / (k1_ms * 1e-3) / 1e9
    it_gbs = it_bytes / (it_ms * 1e-3) / 1e9
    stored_cap = peak * 1e9 / 136 / 1e9  # GDOF/s at the stored-geometry HBM bound
    return {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic,
            "traffic_ncu": "profiles/k1_traffic.json (ncu --set full dram bytes per K1 launch)",
            "geometry": geo,
            "algorithmic_bytes_per_node": k1_bytes / nodes, "k1_ms": k1_ms, "k2_ms": k2_ms,
            "k1_share": k1_ms / max(k1_ms + k2_ms, 1e-12),
            "iteration": {"bytes_per_node": it_bytes / nodes, "achieved_gbs": it_gbs,
                          "frac": it_gbs / peak,
                          "stored_geometry_bound_gdofs": stored_cap}}


def ax_microbench(peak, reps=10):
    """BASELINE configs[1] / SURVEY C2: the standalone Helmholtz Ax (h1 = h2 = 1)
    on a 32^3 N=7 deformed box, 1 GPU, u ~ U(-1,1); 1 warm-up + reps, min and
    median; roofline from 72 algorithmic B/node (u, g1..g6, bm read; w written)."""
    import torch

    import paper_2109_03592_b200 as sb
    ctx = sb.Context.box(32, 32, 32, 7, deform=0.05, device=0)
    g = torch.Generator(device="cuda:0").manual_seed(1)
    u = torch.rand(ctx.nodes, dtype=torch.float64, device="cuda:0", generator=g) * 2 - 1
    w = torch.empty_like(u)
    co = sb.HelmholtzCoeffs(1.0, 1.0)
    sb.axhelm(u, co, ctx, out=w)
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sb.axhelm(u, co, ctx, out=w)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    nodes = ctx.nodes
    ctx.close()
    tmin, tmed = min(ts), statistics.median(ts)
    gbs = 72 * nodes / (tmin * 1e-3) / 1e9
    return {"config": "Helmholtz Ax h1=h2=1, 32^3 N=7 deformed box, 1 GPU (BASELINE configs[1])",
            "ms_min": tmin, "ms_median": tmed, "gdofs": nodes / (tmin * 1e-3) / 1e9,
            "kernel": ("ax_tma_kernel (FMA)" if os.environ.get("SBX_K1_FMA") else
                       "ax_dmma_kernel (FP64 tensor cores, stored G)"),
            "algorithmic_bytes_per_node": 72, "achieved_gbs": gbs, "peak": peak,
            "frac": gbs / peak}


def bench_config(ex, ey, ez, N, iters, world):
    """The workload, identical in both arms (the reference arm times a bounded
    sample of exactly this; its sampling details are in its cpu_baseline)."""
    nodes = ex * ey * ez * (N + 1) ** 3
    return {"workload": "Poisson PCG, Jacobi, deformed box (a=0.05), zero guess",
            "elements": [ex, ey, ez], "degree": N, "local_nodes": nodes,
            "iterations_per_step": iters, "parallelism": f"rcb{world}",
            "l2": (f"inputs larger than L2 (per-iteration working set {nodes * 88.4 / 1e9:.1f} "
                   "GB >> 126 MB)") if nodes * 88.4 > 1e9 else
                  f"working set {nodes * 88.4 / 1e6:.0f} MB: comparable to L2 (not the bench size)"}


def k1_kernel_name(N):
    tc = k1_geometry(N) == "trilinear" and not os.environ.get("SBX_K1_FMA")
    if tc and N == 7:
        return "k1_dmma_kernel (K1 on the FP64 tensor cores: p/x update + axhelm + p'Ap)"
    if tc and N == 9:
        return "k1_dmma10_kernel (K1 on the FP64 tensor cores, whole-element GEMMs)"
    if tc and N in (5, 11) and not os.environ.get("SBX_K1_FMAG"):
        return f"k1_dmmag_kernel<{N + 1}> (K1 on the FP64 tensor cores, whole-element GEMMs)"
    return "ax_tma_kernel (K1: p/x update + axhelm + p'Ap)"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,power.limit")

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.Q}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([s.strip() for s in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        def num(col):
            v = []
            for s in self.samples:
                try:
                    v.append(float(s[col]))
                except (IndexError, ValueError):
                    pass
            return v
        pw, pl = num(6), num(7)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples),
                "power_w": statistics.median(pw) if pw else None,
                "power_limit_w": max(pl) if pl else None}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--elements", type=int, nargs=3, default=[64, 64, 64])
    ap.add_argument("--degree", type=int, default=7)
    ap.add_argument("--iters", type=int, default=100, help="CG iterations per step")
    ap.add_argument("--deform", type=float, default=0.05)
    ap.add_argument("--ref-iters", type=int, default=6,
                    help="reference pcg iterations per timed CPU step (bounded sample)")
    ap.add_argument("--no-one-worker", action="store_true",
                    help="skip the 1-thread reference figure")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ax-microbench", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------- CPU arm --
def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


_REF_PROBLEM = {}


def ref_problem(ex, ey, ez, N, deform):
    """The reference's own problem (oracle/_ref: sembox compiled unmodified;
    the C port if the build is absent), with the benchmark right-hand side
    prepared inside it.  Built once per process (untimed setup)."""
    from oracle import oracle as O

    key = (ex, ey, ez, N, deform)
    if key not in _REF_PROBLEM:
        if not O.ref_available() and os.path.isdir("/root/reference"):
            O.build(ref=True)
        backend = "ref" if O.ref_available() else "port"
        cr = O.box_corners(ex, ey, ez, deform=deform)
        if backend == "ref":
            O._ref().ref_set_workers(os.cpu_count() or 1)
        P = O.Problem(ex, ey, ez, N, corners=cr, backend=backend)
        b = P.rhs_random_continuous(77)
        if backend == "ref":
            P.bench_prepare(b)
            P.drop("inv_mult", "mask")
        _REF_PROBLEM[key] = (P, b, backend)
    return _REF_PROBLEM[key]


def cpu_reference_run(ex, ey, ez, N, deform, iters, steps, warmup, workers=None):
    """Times the reference's pcg (krylov.cpp:7-91 with HelmholtzOperator, the
    parallel Jacobi lambda and the weighted dot) on the SAME mesh as the GPU
    arm, `iters` iterations per step (tolerance 0), with `workers` host
    threads (default: all).  Also times the solve's fixed start-up (a
    0-iteration pcg: b'b, the zero-guess scan, the first preconditioner
    application and dots) so the per-iteration cost can be separated from it.
    Returns (step seconds list, startup seconds, backend, threads, nodes)."""
    from oracle import oracle as O

    P, b, backend = ref_problem(ex, ey, ez, N, deform)
    cores = os.cpu_count() or 1
    threads = workers or cores
    if backend == "ref":
        O._ref().ref_set_workers(threads)

        def solve(k):
            got = P.bench_solve(k)
            assert got == k, (got, k)
    else:
        threads = 1

        def solve(k):
            r = P.pcg(b, 1.0, 0.0, "jacobi", 0.0, k)
            assert r.iterations == k, (r.iterations, k)

    for _ in range(warmup):
        solve(iters)
    t0 = time.perf_counter()
    solve(0)
    startup = time.perf_counter() - t0
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        solve(iters)
        times.append(time.perf_counter() - t0)
    if backend == "ref":
        O._ref().ref_set_workers(cores)
    return times, startup, backend, threads, P.nodes_count


def cpu_summary(times, startup, nodes, iters, full_iters):
    """Per-iteration cost from the timed steps (step - start-up) / iterations,
    and the metric for the benchmark's own step (start-up + full_iters
    iterations), in GDOF/s of local nodes."""
    t = statistics.median(times)
    t_it = max(t - startup, 1e-9) / max(iters, 1)
    full = startup + full_iters * t_it
    return {"value": nodes * full_iters / full / 1e9,
            "sample_value": nodes * iters / t / 1e9,
            "ms_per_iteration": t_it * 1e3, "startup_ms": startup * 1e3,
            "ms_per_sample_step": t * 1e3}


def run_reference_arm(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    ex, ey, ez = args.elements
    N = args.degree
    iters = args.ref_iters
    t_setup = time.perf_counter()
    ref_problem(ex, ey, ez, N, args.deform)
    t_setup = time.perf_counter() - t_setup
    times, startup, backend, cores, nodes = cpu_reference_run(
        ex, ey, ez, N, args.deform, iters, max(args.steps, 1), args.warmup)
    s = cpu_summary(times, startup, nodes, iters, args.iters)
    # one host thread: a bounded 1-iteration sample
    one = None
    if backend == "ref" and not args.no_one_worker:
        t1, st1, _, _, _ = cpu_reference_run(ex, ey, ez, N, args.deform, 1, 1, 0, workers=1)
        one = cpu_summary(t1, st1, nodes, 1, args.iters)
        one["cores"] = 1
    val = s["value"]
    sample = (f"the {ex}x{ey}x{ez} N={N} bench mesh itself (same config as the GPU arm); each "
              f"timed step is a {iters}-iteration reference pcg from x=0 (tol 0); value = "
              f"local nodes x {args.iters} / (start-up + {args.iters} x per-iteration time), "
              f"i.e. the bench's {args.iters}-iteration step, from the measured start-up "
              f"({s['startup_ms']:.0f} ms, a 0-iteration pcg) and the measured per-iteration "
              f"cost ((step - start-up) / {iters})")
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup,
            "ms_per_step": s["startup_ms"] + args.iters * s["ms_per_iteration"],
            "ms_per_iteration": s["ms_per_iteration"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": bench_config(ex, ey, ez, N, args.iters, args.gpus),
            "arm": {"parallelism": f"reference CPU pcg, {cores} host threads",
                    "timed_sample": {"elements": [ex, ey, ez],
                                     "iterations_per_timed_step": iters},
                    "setup_s": round(t_setup, 2)},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores,
                             "kind": "reference" if backend == "ref" else "port",
                             "cpu_model": cpu_model(), "sample": sample,
                             "sample_value": s["sample_value"],
                             "ms_per_iteration": s["ms_per_iteration"],
                             "startup_ms": s["startup_ms"], "one_worker": one},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------- GPU arm --
def run_ours(args):
    import numpy as np
    import torch

    import paper_2109_03592_b200 as sb

    rank, world, local = dist_env()
    if world > 1:
        return run_ours_dist(args)
    torch.cuda.set_device(local)
    ex, ey, ez = args.elements
    N = args.degree
    iters = args.iters
    t_setup = time.perf_counter()
    ctx = sb.Context.box(ex, ey, ez, N, deform=args.deform, device=local)
    t_setup = time.perf_counter() - t_setup
    nodes = ctx.nodes
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    # continuous masked RHS (test_schwarz.cpp:30-38 recipe with a device RNG):
    # random field -> gs_sum -> * inv_mult * mask
    g = torch.Generator(device=f"cuda:{local}").manual_seed(77)
    b = torch.rand(nodes, dtype=torch.float64, device=f"cuda:{local}", generator=g) * 2 - 1
    sb.gs_sum_inplace(ctx, b)
    inv = torch.from_numpy(ctx.array(1)).cuda(local)
    mask = torch.from_numpy(ctx.array(0)).cuda(local)
    b.mul_(inv * mask)
    del inv, mask
    x = torch.zeros_like(b)
    cfg = sb.KrylovConfig(tolerance=0.0, max_iterations=iters)

    def step_dev():
        x.zero_()
        return sb.pcg(op, b, x, cfg, history=False)

    for _ in range(args.warmup):
        r = step_dev()
    assert r.iterations == iters
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step_dev()
        ev1.record()
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    value = nodes * iters / (ms * 1e-3) / 1e9

    # e2e: pinned host b/x through the C ABI, copies inside the timed region
    hb = torch.empty(nodes, dtype=torch.float64, pin_memory=True)
    hb.copy_(b)
    hx = torch.zeros(nodes, dtype=torch.float64, pin_memory=True)

    def step_host():
        hx.zero_()
        return sb.pcg(op, hb, hx, cfg, history=False)

    step_host()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_host()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / args.steps
    e2e_val = nodes * iters / (e2e_ms * 1e-3) / 1e9

    # per-kernel device time (timing mode: same kernels, host-launched, events
    # on the launching stream) -> roofline of the dominant kernel
    ctx.enable_timing(True)
    x.zero_()
    sb.pcg(op, b, x, cfg, history=False)
    ctx.enable_timing(False)
    ax_ms, ax_n = ctx.kernel_time("ax")
    up_ms, up_n = ctx.kernel_time("update")
    peak, peak_kind = load_peaks()
    k1_ms = ax_ms / max(ax_n, 1)
    k2_ms = up_ms / max(up_n, 1)
    # DRAM bytes are not measurable in-run without a profiler: traffic stays
    # null here; the ncu capture of the same kernels is under profiles/
    traffic = None

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "ms_per_iteration": ms / iters,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": bench_config(ex, ey, ez, N, iters, 1),
            "arm": {"parallelism": "one B200, FAST solver (one CUDA graph per solve)",
                    "setup_s": round(t_setup, 2)},
            "e2e": {"value": e2e_val, "unit": UNIT, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 2 * 8 * nodes, "d2h_bytes_per_step": 8 * nodes},
            # per solve: rhs check, prologue, 2 per iteration (K1, K2), final update
            "gpu_launches": args.steps * (2 * iters + 3),
            "roofline": roofline_block(N, ex * ey * ez, nodes, k1_ms, k2_ms, ms / iters, peak,
                                       peak_kind, traffic, k1_kernel_name(N)),
            "clocks": clk.summary()}
    line["unique_dof_gdofs"] = value * unique_fraction(ex, ey, ez, N)
    if not args.no_ax_microbench:
        line["ax_microbench"] = ax_microbench(peak)
    if not args.no_cpu_baseline:
        # the reference pcg on this box's host cores, same mesh, bounded sample
        times, startup, backend, cores, cnodes = cpu_reference_run(
            ex, ey, ez, N, args.deform, args.ref_iters, 1, 0)
        cs = cpu_summary(times, startup, cnodes, args.ref_iters, iters)
        line["cpu_baseline"] = {
            "value": cs["value"], "unit": UNIT, "cores": cores,
            "kind": "reference" if backend == "ref" else "port", "cpu_model": cpu_model(),
            "sample": f"{ex}x{ey}x{ez} N={N} (the bench mesh), one {args.ref_iters}-iteration "
                      f"reference pcg after a 0-iteration start-up probe; value projected to "
                      f"the {iters}-iteration step (see --impl reference)",
            "ms_per_iteration": cs["ms_per_iteration"], "startup_ms": cs["startup_ms"]}
        _REF_PROBLEM.clear()
    print(json.dumps(line), flush=True)


def run_ours_dist(args):
    """N > 1: the same workload partitioned by RCB over the ranks (strong
    scaling); one process per GPU, peer-window exchanges inside the solve."""
    import torch
    import torch.distributed as dist

    import paper_2109_03592_b200 as sb
    from paper_2109_03592_b200.dist import DistContext

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    ex, ey, ez = args.elements
    N = args.degree
    iters = args.iters
    t_setup = time.perf_counter()
    ctx = DistContext.box(ex, ey, ez, N, deform=args.deform, device=local)
    t_setup = time.perf_counter() - t_setup
    nodes_global = ex * ey * ez * (N + 1) ** 3
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    g = torch.Generator(device=f"cuda:{local}").manual_seed(77 + rank)
    b = torch.rand(ctx.nodes, dtype=torch.float64, device=f"cuda:{local}", generator=g) * 2 - 1
    sb.gs_sum_inplace(ctx, b)  # distributed gather-scatter: continuous across ranks
    inv = torch.from_numpy(ctx.array(1)).cuda(local)
    mask = torch.from_numpy(ctx.array(0)).cuda(local)
    b.mul_(inv * mask)
    del inv, mask
    x = torch.zeros_like(b)
    cfg = sb.KrylovConfig(tolerance=0.0, max_iterations=iters)

    def step():
        x.zero_()
        return sb.pcg(op, b, x, cfg, history=False)

    for _ in range(args.warmup):
        r = step()
    assert r.iterations == iters
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
        dist.barrier()
    ms_local = ev0.elapsed_time(ev1) / args.steps
    t = torch.tensor([ms_local], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = nodes_global * iters / (ms * 1e-3) / 1e9
    # e2e: each rank's b/x from pinned host memory through the C ABI
    hb = torch.empty(ctx.nodes, dtype=torch.float64, pin_memory=True)
    hb.copy_(b)
    hx = torch.zeros(ctx.nodes, dtype=torch.float64, pin_memory=True)

    def step_host():
        hx.zero_()
        return sb.pcg(op, hb, hx, cfg, history=False)

    step_host()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step_host()
    e2e_local = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([e2e_local], dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())
    # per-kernel times (timing mode; every rank takes part in the exchanges);
    # skipped under SBX_TRACE so the device trace keeps the graph-mode solve
    ax_ms = up_ms = float("nan")
    ax_n = up_n = 1
    if not (os.environ.get("SBX_TRACE") or os.environ.get("SBX_TRACE1")):
        ctx.enable_timing(True)
        x.zero_()
        sb.pcg(op, b, x, cfg, history=False)
        ctx.enable_timing(False)
        ax_ms, ax_n = ctx.kernel_time("ax")
        up_ms, up_n = ctx.kernel_time("update")
    peak, peak_kind = load_peaks()
    clocks = clk.summary()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                "ms_per_iteration": ms / iters, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": bench_config(ex, ey, ez, N, iters, world),
                "arm": {"parallelism": f"rcb{world}: elements partitioned, peer-window halo "
                                       "+ scalar exchange over NVLink",
                        "elements_per_rank": ctx.elem_count, "setup_s": round(t_setup, 2)},
                "e2e": {"value": nodes_global * iters / (e2e_ms * 1e-3) / 1e9, "unit": UNIT,
                        "ms_per_step": e2e_ms, "h2d_bytes_per_step": 2 * 8 * nodes_global,
                        "d2h_bytes_per_step": 8 * nodes_global},
                "gpu_launches": args.steps * (3 * iters + 6) * world,
                "roofline": roofline_block(N, ctx.elem_count, ctx.nodes,
                                           ax_ms / max(ax_n, 1), up_ms / max(up_n, 1),
                                           ms / iters, peak, peak_kind, None,
                                           k1_kernel_name(N) + " on rank 0; k2_ms = halo "
                                           "assembly + K2 + scalar exchange"),
                "clocks": clocks,
                "unique_dof_gdofs": value * unique_fraction(ex, ey, ez, N)}
        print(json.dumps(line), flush=True)
    ctx.close()
    dist.barrier()
    dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
