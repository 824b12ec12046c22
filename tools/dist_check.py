"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --standalone --nproc-per-node 2 tools/dist_check.py

Per rank: distributed context of a deformed box; compares with the
single-process reference (oracle) restricted to the rank's elements:
  * gather-scatter and the assembled operator: bitwise (canonical copy order);
  * PCG (FAST): same iteration count as the reference, solution within 1e-10.
Prints one line per rank, exits non-zero on any mismatch.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SBX_OVERSUB=1: more ranks than GPUs (rank r on GPU r % count; the blob
    # exchange then runs over gloo, since NCCL refuses two ranks per GPU) --
    # exercises the 8-rank exchange logic on a 4-GPU box
    if os.environ.get("SBX_OVERSUB"):
        local = local % torch.cuda.device_count()
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")
    else:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    rank, world = dist.get_rank(), dist.get_world_size()
    import paper_2109_03592_b200 as sb
    from oracle import oracle as O
    from paper_2109_03592_b200.dist import DistContext

    failures = []
    F = (False, False, False)
    cases = [(8, 8, 8, 7, 0.05, 1e-8, F, 0.0), (6, 5, 4, 5, 0.03, 1e-10, F, 0.0),
             # periodic in x and z (Dirichlet only on the y faces), Helmholtz
             (6, 4, 4, 7, 0.0, 1e-10, (True, False, True), 1.0)]
    for (ex, ey, ez, N, deform, tol, per, h2) in cases:
        ctx = DistContext.box(ex, ey, ez, N, deform=deform, periodic=per, device=local)
        mesh = sb.build_box_mesh(ex, ey, ez, periodic=per, deform=deform)
        G = O.Problem(ex, ey, ez, N, periodic=per, corners=mesh.corners)
        n3 = (N + 1) ** 3
        ln = (ctx.local_elements[:, None] * n3 + np.arange(n3)[None, :]).ravel()
        f = O.fill_uniform(99, G.nodes_count)
        ref = f.copy()
        G.gs_sum_inplace(ref)
        got = sb.gs_sum(ctx, torch.from_numpy(f[ln]).cuda())
        if not np.array_equal(got.cpu().numpy(), ref[ln]):
            failures.append(f"gs {ex}x{ey}x{ez} N={N}")
        # assembled operator (fast kernels: tolerance), masked
        op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, h2))
        u = G.rhs_random_continuous(5)
        q = torch.empty(ln.size, dtype=torch.float64, device="cuda")
        op.apply(torch.from_numpy(u[ln]).cuda(), q)
        qa = G.apply(u, 1.0, h2)[ln]
        err = np.linalg.norm(q.cpu().numpy() - qa) / np.linalg.norm(qa)
        if not err <= 1e-12:
            failures.append(f"apply rel err {err:.2e}")
        # PCG
        b = G.rhs_random_continuous(77)
        refp = G.pcg(b, 1.0, h2, "jacobi", tol, 5000)
        x = torch.zeros(ln.size, dtype=torch.float64, device="cuda")
        r = sb.pcg(op, torch.from_numpy(b[ln]).cuda(), x, sb.KrylovConfig(tol, 5000))
        xe = np.linalg.norm(x.cpu().numpy() - refp.x[ln]) / max(np.linalg.norm(refp.x[ln]), 1e-300)
        ok = r.iterations == refp.iterations and xe <= 1e-10 and r.converged
        if not ok:
            failures.append(f"pcg its {r.iterations} vs {refp.iterations}, x err {xe:.2e}")
        print(f"rank {rank}/{world} box {ex}x{ey}x{ez} N={N} per={per} h2={h2}: "
              f"{ctx.elem_count} elements, "
              f"pcg {r.iterations} its (ref {refp.iterations}), x err {xe:.2e}, apply err "
              f"{err:.2e}", flush=True)
        ctx.close()
    dist.barrier()
    dist.destroy_process_group()
    if failures:
        print(f"rank {rank} FAILURES: {failures}", flush=True)
        sys.exit(1)
    print(f"rank {rank} ALL OK", flush=True)


if __name__ == "__main__":
    main()
