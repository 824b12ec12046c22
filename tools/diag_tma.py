"""Diagnose the TMA K1 path: repeated solves at growing sizes."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2109_03592_b200 as sb
its = int(os.environ.get("ITS", "50"))
torch.manual_seed(0)
for m in [int(a) for a in sys.argv[1:]]:
    ctx = sb.Context.box(m, m, m, 7, deform=0.05)
    b = torch.rand(ctx.nodes, dtype=torch.float64, device="cuda")
    sb.gs_sum_inplace(ctx, b)
    b.mul_(torch.from_numpy(ctx.array(1) * ctx.array(0)).cuda())
    x = torch.zeros_like(b)
    op = sb.HelmholtzOperator(ctx)
    for rep in range(3):
        t = time.time()
        try:
            x.zero_()
            r = sb.pcg(op, b, x, sb.KrylovConfig(0.0, its), history=False)
            torch.cuda.synchronize()
            print(m, rep, "ok", r.iterations, r.rel_residual, f"{time.time()-t:.3f}s", flush=True)
        except Exception as e:
            print(m, rep, "FAIL", e, flush=True)
            sys.exit(1)
    ctx.enable_timing(True)
    x.zero_()
    r = sb.pcg(op, b, x, sb.KrylovConfig(0.0, its), history=False)
    print(m, "timing ok", ctx.kernel_time("ax"), ctx.kernel_time("update"), flush=True)
