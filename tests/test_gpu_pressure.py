"""The consistent-Poisson pressure path (pressure.cu)
against the UNMODIFIED reference (oracle/_ref): gradient_from_pressure and
divergence_to_pressure (operators.cpp:327-410), FlowSolver's
apply_pressure_operator and pressure_operator_diagonal (stepper.cpp:240-275,
restated in oracle/ref_shim.cpp with the reference's own operators), and the
pressure PCG of solve_pressure_update (stepper.cpp:277-348: Jacobi or none,
mean deflation, plain dot).

* EXACT mode (the reference's evaluation order): every operator bitwise, the
  PCG residual history and solution bit for bit.
* FAST mode (fused kernels): operators within 1e-12 relative L2; the PCG
  tracks the reference history while round-off is small, and a converged
  solve lands on the same solution.  (The pressure CG amplifies last-digit
  differences quickly -- the histories drift apart by ~1e-6 after ~60
  iterations (profiles/r02_pressure.md) -- so equal iteration counts at a
  tolerance are a property of the EXACT mode.)"""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

OP_TOL = 1e-12
FINAL_TOL = 1e-10


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def refready():
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")


def make(dims, N, deform, periodic=(False, False, False)):
    ctx = sb.Context.box(*dims, N, periodic=periodic, deform=deform)
    P = O.Problem(*dims, N, periodic=periodic,
                  corners=O.box_corners(*dims, deform=deform), backend="ref")
    P.pressure_setup()
    return ctx, P


CASES = [((3, 2, 2), 3, 0.05, (False,) * 3), ((2, 2, 3), 4, 0.04, (False,) * 3),
         ((3, 3, 2), 5, 0.05, (False,) * 3), ((3, 2, 2), 7, 0.05, (False,) * 3),
         ((2, 3, 2), 7, 0.03, (True, False, False)), ((2, 2, 2), 9, 0.05, (False,) * 3),
         ((2, 2, 1), 12, 0.02, (False,) * 3), ((1, 2, 2), 15, 0.02, (False,) * 3)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c[1]}")
def test_pressure_operators(cuda, refready, case):
    torch = cuda
    dims, N, deform, per = case
    ctx, P = make(dims, N, deform, per)
    p = O.fill_uniform(60 + N, P.pnodes_count)
    # gradient (velocity grid, three components)
    want = P.gradient_from_pressure(p)
    got = sb.gradient_from_pressure(p, ctx)
    for c in range(3):
        assert rel(got[c], want[c]) <= OP_TOL, ("grad", c, rel(got[c], want[c]))
    # device tensors give the same bits as host arrays
    gd = sb.gradient_from_pressure(torch.from_numpy(p).cuda(), ctx)
    for c in range(3):
        assert np.array_equal(gd[c].cpu().numpy(), got[c])
    # divergence of a random velocity field
    u = [O.fill_uniform(70 + N + c, P.nodes_count) for c in range(3)]
    assert rel(sb.divergence_to_pressure(*u, ctx), P.divergence_to_pressure(*u)) <= OP_TOL
    # the assembled pressure operator and its diagonal
    E = sb.PressureOperator(ctx)
    q = np.empty_like(p)
    E.apply(p, q)
    assert rel(q, P.pressure_apply(p)) <= OP_TOL
    d = E.diagonal()
    dref = P.pressure_array(6)
    assert np.max(np.abs(d - dref) / np.abs(dref)) <= OP_TOL
    # EXACT: the reference's bits
    ge = sb.gradient_from_pressure(p, ctx, exact=True)
    for c in range(3):
        assert np.array_equal(ge[c], want[c]), ("grad exact", c)
    assert np.array_equal(sb.divergence_to_pressure(*u, ctx, exact=True),
                          P.divergence_to_pressure(*u))
    Ex = sb.PressureOperator(ctx, exact=True)
    qx = np.empty_like(p)
    Ex.apply(p, qx)
    assert np.array_equal(qx, P.pressure_apply(p))
    if N <= 9:  # the exact diagonal is O(m^3) gradients per element
        assert np.array_equal(Ex.diagonal(), dref)
    # symmetric under the plain dot (Div is the exact transpose of Grad)
    p2 = O.fill_uniform(90 + N, P.pnodes_count)
    q2 = np.empty_like(p2)
    E.apply(p2, q2)
    assert abs(p2 @ q - p @ q2) <= 1e-11 * abs(p @ q2)
    ctx.close()


PCG_CASES = [((3, 3, 3), 5, 0.05), ((3, 3, 2), 7, 0.05), ((2, 2, 2), 9, 0.04)]


@pytest.mark.parametrize("case", PCG_CASES, ids=lambda c: f"N{c[1]}")
@pytest.mark.parametrize("precond", ["jacobi", "none"])
def test_pressure_pcg_exact_bitwise(cuda, refready, case, precond):
    dims, N, deform = case
    ctx, P = make(dims, N, deform)
    b = P.pressure_rhs(5)
    E = sb.PressureOperator(ctx, exact=True)
    for tol, x0 in ((1e-8, None), (1e-10, 0.3)):
        xin = None if x0 is None else x0 * P.pressure_rhs(11)
        ref = P.pressure_pcg(b, precond, tol, 5000, x0=xin)
        assert ref.status == 0 and ref.converged
        x = np.zeros_like(b) if xin is None else xin.copy()
        r = sb.pcg_pressure(E, b, x, sb.KrylovConfig(tol, 5000), precond=precond, mode="exact")
        assert r.iterations == ref.iterations
        assert np.array_equal(np.asarray(r.residual_history), ref.residual_history)
        assert np.array_equal(x, ref.x)
        assert r.rel_residual == ref.rel_residual
    ctx.close()


@pytest.mark.parametrize("case", PCG_CASES, ids=lambda c: f"N{c[1]}")
@pytest.mark.parametrize("precond", ["jacobi", "none"])
def test_pressure_pcg_fast(cuda, refready, case, precond):
    dims, N, deform = case
    ctx, P = make(dims, N, deform)
    b = P.pressure_rhs(5)
    E = sb.PressureOperator(ctx)
    # the early history, while round-off is small, to 1e-9 relative
    ref = P.pressure_pcg(b, precond, 0.0, 30)
    x = np.zeros_like(b)
    r = sb.pcg_pressure(E, b, x, sb.KrylovConfig(0.0, 30), precond=precond)
    np.testing.assert_allclose(r.residual_history, ref.residual_history, rtol=1e-9)
    assert rel(x, ref.x) <= 1e-9
    # converged solves (the reference's default pressure tolerance 1e-6 and a
    # tight one): the same solution, iteration counts within a few percent
    for tol in (1e-6, 1e-10):
        ref = P.pressure_pcg(b, precond, tol, 5000)
        x = np.zeros_like(b)
        r = sb.pcg_pressure(E, b, x, sb.KrylovConfig(tol, 5000), precond=precond)
        assert r.converged and ref.converged
        assert abs(r.iterations - ref.iterations) <= max(3, ref.iterations // 20), (
            r.iterations, ref.iterations)
        assert r.rel_residual <= tol and r.rel_residual_precond <= tol
        assert rel(x, ref.x) <= 100 * tol, rel(x, ref.x)
    # nonzero initial guess (projection-style): r = b - E x0
    x0 = 0.5 * ref.x
    ref2 = P.pressure_pcg(b, precond, 1e-10, 5000, x0=x0)
    x2 = x0.copy()
    r2 = sb.pcg_pressure(E, b, x2, sb.KrylovConfig(1e-10, 5000), precond=precond)
    assert abs(r2.iterations - ref2.iterations) <= max(3, ref2.iterations // 20)
    assert rel(x2, ref2.x) <= 1e-8
    ctx.close()


def test_pressure_errors(cuda):
    ctx = sb.Context.box(2, 2, 2, 2)
    with pytest.raises(sb.ConfigError):
        sb.PressureOperator(ctx)
    ctx.close()
    mesh = sb.build_box_mesh(2, 2, 2, deform=0.05)
    basis = sb.build_gll_basis(5)
    plain = sb.Context.from_problem(sb.build_geometric_factors(mesh, basis), basis,
                                    sb.build_gather_scatter(mesh, 5),
                                    sb.build_dirichlet_mask(mesh, 5))
    with pytest.raises(sb.ConfigError):
        sb.PressureOperator(plain)  # no element corners: no GL metric
    hinted = sb.Context.from_problem(sb.build_geometric_factors(mesh, basis), basis,
                                     sb.build_gather_scatter(mesh, 5),
                                     sb.build_dirichlet_mask(mesh, 5), mesh=mesh)
    assert sb.PressureOperator(hinted).nodes == 8 * 4 ** 3
    with pytest.raises(sb.ConfigError):
        sb.build_pressure_basis(2)
