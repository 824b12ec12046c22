"""Timing of the SURVEY 8(f) rows on one B200 (diagnostics; the headline
metric is bench.py): the batched 3-component velocity solve, the FAST
pressure PCG, the pressure operator's kernels, advection and the projection
history, on a deformed box (default 64^3, N=7).  CUDA events on the current
stream after warm-up; one JSON line per item.

    python tools/flow_bench.py [ex ey ez] [N]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03592_b200 as sb  # noqa: E402


def timed(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def main():
    dims = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else [64, 64, 64]
    N = int(sys.argv[4]) if len(sys.argv) > 4 else 7
    torch.cuda.set_device(0)
    ctx = sb.Context.box(*dims, N, deform=0.05)
    nodes = ctx.nodes
    g = torch.Generator(device="cuda").manual_seed(3)

    def cont(seed):  # continuous masked velocity-grid field
        f = torch.rand(nodes, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
        sb.gs_sum_inplace(ctx, f)
        return f * torch.from_numpy(ctx.array(1) * ctx.array(0)).cuda()

    out = {"mesh": dims, "degree": N, "local_nodes": nodes}
    # --- batched velocity solve (Re = 100, dt = 1e-3, BDF2: h2 = 1.5 / dt)
    co = sb.HelmholtzCoeffs(0.01, 1.5e3)
    op = sb.HelmholtzOperator(ctx, co)
    bs = [cont(d) for d in range(3)]
    x0 = [cont(10 + d) for d in range(3)]
    xs = [torch.empty_like(b) for b in bs]
    cfg = sb.KrylovConfig(1e-8, 500)

    def multi():
        for d in range(3):
            xs[d].copy_(x0[d])
        return sb.pcg_multi(op, bs, xs, cfg, history=False)

    def single():
        r = []
        for d in range(3):
            xs[d].copy_(x0[d])
            r.append(sb.pcg(op, bs[d], xs[d], cfg, history=False))
        return r

    ms_m, rm = timed(multi)
    ms_s, rs = timed(single)
    its = [r.iterations for r in rm]
    out["velocity_batched"] = {"ms": ms_m, "iterations": its, "ms_three_single_solves": ms_s,
                               "gdofs": nodes * sum(its) / (ms_m * 1e-3) / 1e9}
    # --- per-solve overhead: a 20-iteration Poisson solve against 20 iterations
    # of a 100-iteration one (the difference is the prologue + final update)
    opp = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    xp = torch.zeros_like(bs[0])

    def solve(k):
        xp.zero_()
        return sb.pcg(opp, bs[0], xp, sb.KrylovConfig(0.0, k), history=False)

    ms20, _ = timed(lambda: solve(20))
    ms100, _ = timed(lambda: solve(100), reps=3)
    per_it = (ms100 - ms20) / 80
    out["per_solve_overhead"] = {"ms_20_iterations": ms20, "ms_100_iterations": ms100,
                                 "ms_per_iteration": per_it,
                                 "outside_iterations_ms": ms20 - 20 * per_it,
                                 "fraction_of_20_iteration_solve": (ms20 - 20 * per_it) / ms20}
    # --- pressure
    E = sb.PressureOperator(ctx)
    Np = E.nodes
    p = torch.rand(Np, dtype=torch.float64, device="cuda", generator=g)
    q = torch.empty_like(p)
    ms_apply, _ = timed(lambda: E.apply(p, q))
    ms_grad, gr = timed(lambda: sb.gradient_from_pressure(p, ctx))
    ms_div, _ = timed(lambda: sb.divergence_to_pressure(*gr, ctx))
    b = sb.divergence_to_pressure(*[cont(20 + d) for d in range(3)], ctx)
    b -= b.mean()
    x = torch.zeros_like(b)
    iters = 50
    pcfg = sb.KrylovConfig(0.0, iters)

    def psolve():
        x.zero_()
        return sb.pcg_pressure(E, b, x, pcfg, history=False)

    ms_p, rp = timed(psolve, reps=3, warm=1)
    out["pressure"] = {"pressure_nodes": Np, "ms_apply": ms_apply, "ms_gradient": ms_grad,
                       "ms_divergence": ms_div, "pcg_iterations": rp.iterations,
                       "pcg_ms_per_iteration": ms_p / iters,
                       "pcg_gdofs_pressure_nodes": Np * iters / (ms_p * 1e-3) / 1e9}
    # --- projection (depth 5) on the pressure solution
    H = sb.ProjectionHistory(ctx, 5)
    for k in range(5):
        H.append(x * (1.0 + 0.1 * k) + 0.01 * k * b)
    ms_guess, _ = timed(lambda: H.project_guess(b))
    out["projection"] = {"depth": H.size(), "ms_guess": ms_guess}
    # --- advection
    u = [cont(30 + d) for d in range(3)]
    ms_adv, _ = timed(lambda: sb.advect(u, u, ctx))
    out["advect"] = {"ms": ms_adv, "bytes_per_node": 80,
                     "achieved_gbs": 80 * nodes / (ms_adv * 1e-3) / 1e9}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
