"""Full-size parity through size-independent properties: the bench workload
(BASELINE.json configs[1]: 64^3 elements, N=7, deformed box a=0.05, 134M local
nodes) is too large for the oracle, so the fused FAST solver is checked against
the separately launched operator kernels (axhelm + gs + mask, sbx_apply) on a
manufactured solution:
  * b = A x*, solve, x ~ x*, and the true residual |b - Ax| agrees with the
    converged recurrence (krylov.cpp:51-57 tests the recurrence only);
  * exact x2 scaling of A, and symmetry <Ax, y> = <x, Ay> (test_operators.cpp:161-171,
    326-348 at full size);
  * a second solve gives identical bits (graph replay, fixed summation trees)."""
import pytest

import paper_2109_03592_b200 as sb

pytestmark = pytest.mark.gpu

TOL = 1e-10          # solver tolerance (relative residual)
TRUE_RES_TOL = 1e-9  # true residual, recomputed outside the solver (B200: 1.0e-10)
ERR_TOL = 1e-5       # |x - x*| / |x*| (B200: 1.7e-7 after 1704 iterations)


def _continuous(ctx, torch, seed, inv, mask):
    g = torch.Generator(device="cuda:0").manual_seed(seed)
    f = torch.rand(ctx.nodes, dtype=torch.float64, device="cuda:0", generator=g) * 2 - 1
    sb.gs_sum_inplace(ctx, f)
    return f.mul_(inv * mask)


def test_fullsize_manufactured_solution(cuda):
    torch = cuda
    ctx = sb.Context.box(64, 64, 64, 7, deform=0.05, device=0)
    inv = torch.from_numpy(ctx.array(1)).cuda()
    mask = torch.from_numpy(ctx.array(0)).cuda()
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    xs = _continuous(ctx, torch, 5, inv, mask)
    y = _continuous(ctx, torch, 6, inv, mask)

    ax, ay = torch.empty_like(xs), torch.empty_like(xs)
    op.apply(xs, ax)
    op.apply(y, ay)
    a2 = torch.empty_like(xs)
    op.apply(2 * xs, a2)
    assert torch.equal(a2, 2 * ax)
    w = inv  # continuous fields: the unique-DOF inner product is sum(u v / mult)
    lhs, rhs = float((ax * y * w).sum()), float((xs * ay * w).sum())
    assert abs(lhs - rhs) <= 1e-11 * abs(rhs)
    assert float((ax * xs * w).sum()) > 0

    b = ax
    x = torch.zeros_like(b)
    r = sb.pcg(op, b, x, sb.KrylovConfig(TOL, 5000), history=False)
    assert r.converged and 0 < r.iterations < 5000
    res = torch.empty_like(b)
    op.apply(x, res)
    true_rel = float(torch.linalg.vector_norm(b - res) / torch.linalg.vector_norm(b))
    assert true_rel <= TRUE_RES_TOL, true_rel
    err = float(torch.linalg.vector_norm(x - xs) / torch.linalg.vector_norm(xs))
    print(f"64^3 N=7: {r.iterations} iterations, true rel. residual {true_rel:.3e}, error {err:.3e}")
    assert err <= ERR_TOL, err

    x2 = torch.zeros_like(b)
    r2 = sb.pcg(op, b, x2, sb.KrylovConfig(TOL, 5000), history=False)
    assert r2.iterations == r.iterations and torch.equal(x2, x)
