"""Timing probe: K1 / iteration time of the same 1-GPU problem through the
single-GPU context and through a 1-rank distributed context (diagnostics)."""
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2109_03592_b200 as sb  # noqa: E402
from paper_2109_03592_b200.dist import DistContext  # noqa: E402


def measure(ctx, label, iters=100):
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    g = torch.Generator(device="cuda:0").manual_seed(77)
    b = torch.rand(ctx.nodes, dtype=torch.float64, device="cuda:0", generator=g) * 2 - 1
    sb.gs_sum_inplace(ctx, b)
    inv = torch.from_numpy(ctx.array(1)).cuda(0)
    mask = torch.from_numpy(ctx.array(0)).cuda(0)
    b.mul_(inv * mask)
    x = torch.zeros_like(b)
    cfg = sb.KrylovConfig(tolerance=0.0, max_iterations=iters)
    for _ in range(3):
        x.zero_()
        sb.pcg(op, b, x, cfg, history=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        x.zero_()
        sb.pcg(op, b, x, cfg, history=False)
    e1.record()
    torch.cuda.synchronize()
    it_us = e0.elapsed_time(e1) / 5 / iters * 1e3
    ctx.enable_timing(True)
    x.zero_()
    sb.pcg(op, b, x, cfg, history=False)
    ctx.enable_timing(False)
    ax_ms, ax_n = ctx.kernel_time("ax")
    up_ms, up_n = ctx.kernel_time("update")
    print(json.dumps({"case": label, "us_per_it": it_us, "k1_us": ax_ms / ax_n * 1e3,
                      "tail_us": up_ms / up_n * 1e3}), flush=True)


def main():
    E = [int(v) for v in sys.argv[1:4]] if len(sys.argv) > 3 else [32, 32, 16]
    torch.cuda.set_device(0)
    measure(sb.Context.box(*E, 7, deform=0.05, device=0), "plain")
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    measure(sb.Context.box(*E, 7, deform=0.05, device=0), "plain+nccl")
    measure(DistContext.box(*E, 7, deform=0.05, device=0), "dist1")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
