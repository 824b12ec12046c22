"""CUDA operators (libsbx.so, sm_100a) against the oracle: EXACT variants
bitwise, FAST variants within the north-star tolerance (1e-12 relative L2)."""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

AX_TOL = 1e-12  # north_star: Ax within 1e-12 relative L2 in FP64


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def make(ex, ey, ez, N, periodic=(False, False, False), deform=0.0, lengths=(1.0, 1.0, 1.0)):
    mesh = sb.build_box_mesh(ex, ey, ez, lengths=lengths, periodic=periodic, deform=deform)
    basis = sb.build_gll_basis(N)
    gf = sb.build_geometric_factors(mesh, basis)
    gmap = sb.build_gather_scatter(mesh, N)
    mask = sb.build_dirichlet_mask(mesh, N)
    ctx = sb.Context.from_problem(gf, basis, gmap, mask)
    P = O.Problem(ex, ey, ez, N, periodic=periodic, lengths=lengths, corners=mesh.corners)
    return ctx, P


CASES = [(2, 1, 1, 1, (False,) * 3, 0.0), (2, 1, 1, 2, (False,) * 3, 0.0),
         (2, 1, 1, 3, (False,) * 3, 0.0), (2, 2, 1, 4, (True, False, False), 0.0),
         (3, 2, 2, 5, (False,) * 3, 0.05), (2, 2, 2, 6, (False, True, False), 0.03),
         (4, 3, 2, 7, (False,) * 3, 0.05), (2, 2, 2, 8, (True, True, True), 0.0),
         (2, 2, 2, 9, (False,) * 3, 0.05), (2, 1, 2, 10, (False,) * 3, 0.0),
         (1, 1, 2, 15, (False,) * 3, 0.02), (1, 1, 1, 17, (False,) * 3, 0.0)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c[3]}")
def test_axhelm_exact_bitwise_and_fast_tol(cuda, case):
    ex, ey, ez, N, per, deform = case
    ctx, P = make(ex, ey, ez, N, per, deform)
    u = O.fill_uniform(100 + N, P.nodes_count)
    for h1, h2 in ((0.9, 0.4), (1.0, 0.0), (1.0, 1.0)):
        ref = P.axhelm(u, h1, h2)
        got = sb.axhelm(u, sb.HelmholtzCoeffs(h1, h2), ctx, exact=True)
        assert np.array_equal(got, ref), (h1, h2)
        fast = sb.axhelm(u, sb.HelmholtzCoeffs(h1, h2), ctx)
        assert rel_l2(fast, ref) <= AX_TOL
    # mutation hook (operators.cpp:221-222,255): flipped t-term must differ
    flip = sb.axhelm(u, sb.HelmholtzCoeffs(1.0, 0.0), ctx, exact=True, flip=True)
    assert np.array_equal(flip, P.axhelm(u, 1.0, 0.0, flip=True))
    assert rel_l2(flip, P.axhelm(u, 1.0, 0.0)) > 1e-3
    fflip = sb.axhelm(u, sb.HelmholtzCoeffs(1.0, 0.0), ctx, flip=True)
    assert rel_l2(fflip, flip) <= AX_TOL


@pytest.mark.parametrize("case", CASES[:10], ids=lambda c: f"N{c[3]}")
def test_gs_apply_diag_dot_bitwise(cuda, case):
    ex, ey, ez, N, per, deform = case
    ctx, P = make(ex, ey, ez, N, per, deform)
    u = O.fill_uniform(7 + N, P.nodes_count)
    g = u.copy()
    P.gs_sum_inplace(g)
    assert np.array_equal(sb.gs_sum(ctx, u), g)
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(0.5, 2.0), exact=True)
    out = np.empty_like(u)
    op.apply(u, out)
    assert np.array_equal(out, P.apply(u, 0.5, 2.0))
    op_nm = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(0.5, 2.0), use_mask=False, exact=True)
    op_nm.apply(u, out)
    assert np.array_equal(out, P.apply(u, 0.5, 2.0, use_mask=False))
    assert np.array_equal(op.assembled_diagonal(), P.axhelm_diagonal(0.5, 2.0, assembled=True))
    assert sb.field_dot_weighted(ctx, u, g) == P.dot_weighted(u, g)
    fast = sb.field_dot_weighted(ctx, u, g, exact=False)
    assert abs(fast - P.dot_weighted(u, g)) <= 1e-12 * abs(P.dot_weighted(u, g))


def test_golden_operators(cuda, golden):
    for tag in ("ax_a", "ax_b", "ax_c"):
        ex, ey, ez, N = golden[f"{tag}_dims"]
        lengths = tuple(golden[f"{tag}_lengths"])
        ctx, _ = make(ex, ey, ez, N, deform=golden[f"{tag}_deform"][0], lengths=lengths)
        u = golden[f"{tag}_u"]
        assert np.array_equal(sb.axhelm(u, sb.HelmholtzCoeffs(0.9, 0.4), ctx, exact=True),
                              golden[f"{tag}_w"])
        assert np.array_equal(sb.gs_sum(ctx, u), golden[f"{tag}_gs"])
        out = np.empty_like(u)
        sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 1.0), exact=True).apply(u, out)
        assert np.array_equal(out, golden[f"{tag}_apply"])


def test_device_and_host_pointers_agree(cuda):
    torch = cuda
    ctx, P = make(3, 3, 3, 7, deform=0.05)
    u = O.fill_uniform(1, P.nodes_count)
    host = sb.axhelm(u, sb.HelmholtzCoeffs(1.0, 1.0), ctx)
    dev = sb.axhelm(torch.from_numpy(u).cuda(), sb.HelmholtzCoeffs(1.0, 1.0), ctx)
    assert np.array_equal(host, dev.cpu().numpy())


def test_dense_oracle_equivalence(cuda):
    # acceptance.cpp:124-215 / test_operators.cpp:115-144, N <= 4
    for N in (1, 2, 3, 4):
        ctx, P = make(2, 2, 1, N, lengths=(1.2, 0.9, 1.0))
        u = O.fill_uniform(12 + N, P.nodes_count)
        w = sb.axhelm(u, sb.HelmholtzCoeffs(0.7, 1.1), ctx)
        nn = P.nper
        for e in range(P.E):
            A = P.dense_helmholtz_element(e, 0.7, 1.1)
            np.testing.assert_allclose(w[e * nn:(e + 1) * nn], A @ u[e * nn:(e + 1) * nn],
                                       rtol=0, atol=1e-11)


def test_properties(cuda):
    ctx, P = make(2, 2, 2, 3, periodic=(False, True, False))
    # stiffness of constants vanishes; mass-only is exact (test_operators.cpp:122-130)
    ones = np.ones(P.nodes_count)
    assert np.abs(sb.axhelm(ones, sb.HelmholtzCoeffs(1.0, 0.0), ctx)).max() < 1e-12
    u = O.fill_uniform(9, P.nodes_count)
    assert np.array_equal(sb.axhelm(u, sb.HelmholtzCoeffs(0.0, 1.0), ctx, exact=True), P.bm * u)
    # exact x2 scaling (test_operators.cpp:161-171)
    w1 = sb.axhelm(u, sb.HelmholtzCoeffs(1.0, 0.5), ctx)
    w2 = sb.axhelm(2 * u, sb.HelmholtzCoeffs(1.0, 0.5), ctx)
    assert np.array_equal(w2, 2 * w1)
    # assembled operator symmetric positive (test_operators.cpp:326-348)
    x = P.rhs_random_continuous(21)
    y = P.rhs_random_continuous(22)
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 2.0))
    ax, ay = np.empty_like(x), np.empty_like(x)
    op.apply(x, ax)
    op.apply(y, ay)
    lhs, rhs = P.dot_weighted(ax, y), P.dot_weighted(x, ay)
    assert abs(lhs - rhs) <= 1e-11 * abs(rhs)
    assert P.dot_weighted(ax, x) > 0
    # gs(ones) = multiplicity (test_mesh.cpp:117-124)
    assert np.array_equal(sb.gs_sum(ctx, ones), P.mult.astype(float))


def test_shape_errors(cuda):
    ctx, P = make(2, 1, 1, 3)
    with pytest.raises(sb.ContractViolation):
        sb.axhelm(np.zeros(5), sb.HelmholtzCoeffs(), ctx)
    with pytest.raises(sb.ContractViolation):
        sb.gs_sum_inplace(ctx, np.zeros(P.nodes_count + 1))
