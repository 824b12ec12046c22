"""Batched velocity solve: the three component solves of
FlowSolver::solve_velocity_star (stepper.cpp:188-238) -- Helmholtz operator
h1 = 1/Re, h2 = bdf0/dt, Jacobi on its assembled diagonal, the previous
velocity as each component's initial guess -- in one sbx_pcg_multi call
(K1 / K2 once per iteration for all components, grid.y = component).
Against the reference pcg per component (same iteration count, x within
1e-10), and against three separate sbx_pcg calls (the same arithmetic)."""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def velocity_problem(dims, N, deform, seed):
    ctx = sb.Context.box(*dims, N, deform=deform)
    P = O.Problem(*dims, N, corners=O.box_corners(*dims, deform=deform))
    bs = [P.rhs_random_continuous(seed + d) for d in range(3)]
    x0 = [P.rhs_random_continuous(seed + 10 + d) for d in range(3)]  # u_hist[0]
    return ctx, P, bs, x0


@pytest.mark.parametrize("N", [5, 7, 9])
def test_pcg_multi_matches_reference_and_single(cuda, N):
    torch = cuda
    Re, dt, bdf0 = 100.0, 1e-3, 1.5
    co = sb.HelmholtzCoeffs(1.0 / Re, bdf0 / dt)
    ctx, P, bs, x0 = velocity_problem((4, 3, 3), N, 0.05, 31)
    op = sb.HelmholtzOperator(ctx, co)
    tol = 1e-10
    xs = [torch.from_numpy(v.copy()).cuda() for v in x0]
    res = sb.pcg_multi(op, [torch.from_numpy(b).cuda() for b in bs], xs,
                       sb.KrylovConfig(tol, 500))
    for d in range(3):
        ref = P.pcg(bs[d], co.h1, co.h2, "jacobi", tol, 500, x0=x0[d])
        assert res[d].converged and res[d].iterations == ref.iterations, d
        x = xs[d].cpu().numpy()
        assert np.linalg.norm(x - ref.x) / np.linalg.norm(ref.x) <= 1e-10
        # the single solve of the same component: same arithmetic
        xsg = torch.from_numpy(x0[d].copy()).cuda()
        rs = sb.pcg(op, torch.from_numpy(bs[d]).cuda(), xsg, sb.KrylovConfig(tol, 500))
        assert rs.iterations == res[d].iterations
        assert float((xsg - xs[d]).norm() / xsg.norm()) <= 1e-14
    ctx.close()


def test_pcg_multi_mixed_convergence_and_host_buffers(cuda):
    """Components that converge at different iterations (one already at the
    solution, one zero rhs) through host arrays; counts 1 and 2 as well."""
    ctx, P, bs, x0 = velocity_problem((3, 3, 3), 7, 0.04, 5)
    co = sb.HelmholtzCoeffs(0.01, 200.0)
    op = sb.HelmholtzOperator(ctx, co)
    sol = P.pcg(bs[1], co.h1, co.h2, "jacobi", 1e-13, 500).x
    bz = np.zeros_like(bs[2])
    xs = [x0[0].copy(), sol.copy(), x0[2].copy()]
    res = sb.pcg_multi(op, [bs[0], bs[1], bz], xs, sb.KrylovConfig(1e-9, 500))
    ref0 = P.pcg(bs[0], co.h1, co.h2, "jacobi", 1e-9, 500, x0=x0[0])
    ref1 = P.pcg(bs[1], co.h1, co.h2, "jacobi", 1e-9, 500, x0=sol)
    assert res[0].iterations == ref0.iterations
    assert res[1].iterations == ref1.iterations  # 0 or very few
    assert res[2].converged and res[2].iterations == 0 and not xs[2].any()
    assert np.linalg.norm(xs[0] - ref0.x) / np.linalg.norm(ref0.x) <= 1e-10
    for count in (1, 2):
        xs = [v.copy() for v in x0[:count]]
        r = sb.pcg_multi(op, bs[:count], xs, sb.KrylovConfig(1e-9, 500))
        assert [q.iterations for q in r] == [
            P.pcg(bs[d], co.h1, co.h2, "jacobi", 1e-9, 500, x0=x0[d]).iterations
            for d in range(count)]
    # EXACT: the components one after the other, bitwise the reference
    xs = [v.copy() for v in x0]
    r = sb.pcg_multi(op, bs, xs, sb.KrylovConfig(1e-9, 500), mode="exact")
    for d in range(3):
        ref = P.pcg(bs[d], co.h1, co.h2, "jacobi", 1e-9, 500, x0=x0[d])
        assert r[d].iterations == ref.iterations and np.array_equal(xs[d], ref.x)
    ctx.close()
