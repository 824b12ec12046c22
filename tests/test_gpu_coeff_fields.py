"""Per-node Helmholtz coefficients (HelmholtzCoeffs::h1_field / h2_field,
operators.hpp:42-43, read at each node in operators.cpp:242, 258, 292-293)
through sbx_ctx_set_coeff_fields, against the UNMODIFIED reference
(oracle/_ref) with the same fields: axhelm, axhelm_diagonal, apply and the
Jacobi PCG.  With fields the device path evaluates in the reference order in
both modes, so every comparison is bitwise."""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refready():
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")


def fields(P, seed):
    # positive, discontinuous across element faces (the element matrices stay
    # symmetric positive definite; the assembled operator stays SPD)
    h1f = O.fill_uniform(seed, P.nodes_count, 0.5, 2.0)
    h2f = O.fill_uniform(seed + 1, P.nodes_count, 0.0, 3.0)
    return h1f, h2f


CASES = [((3, 2, 2), 5, 0.05), ((2, 2, 2), 7, 0.04), ((2, 2, 1), 8, 0.03)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c[1]}")
def test_operators_with_fields(cuda, refready, case):
    torch = cuda
    dims, N, deform = case
    ctx = sb.Context.box(*dims, N, deform=deform)
    P = O.Problem(*dims, N, corners=O.box_corners(*dims, deform=deform), backend="ref")
    h1f, h2f = fields(P, 40 + N)
    u = O.fill_uniform(50 + N, P.nodes_count)
    for f1, f2 in ((h1f, None), (None, h2f), (h1f, h2f)):
        P.set_coeff_fields(f1, f2)
        co = sb.HelmholtzCoeffs(0.7, 0.3, h1_field=f1, h2_field=f2)
        want = P.axhelm(u, 0.7, 0.3)
        for exact in (True, False):
            assert np.array_equal(sb.axhelm(u, co, ctx, exact=exact), want), (f1 is None, exact)
        # device tensors: the same bits
        cod = sb.HelmholtzCoeffs(0.7, 0.3,
                                 h1_field=None if f1 is None else torch.from_numpy(f1).cuda(),
                                 h2_field=None if f2 is None else torch.from_numpy(f2).cuda())
        got = sb.axhelm(torch.from_numpy(u).cuda(), cod, ctx).cpu().numpy()
        assert np.array_equal(got, want)
        for assembled in (False, True):
            assert np.array_equal(sb.axhelm_diagonal(co, ctx, assembled=assembled),
                                  P.axhelm_diagonal(0.7, 0.3, assembled=assembled))
        q = np.empty_like(u)
        sb.HelmholtzOperator(ctx, co).apply(u, q)
        assert np.array_equal(q, P.apply(u, 0.7, 0.3))
    # the fields apply to one call only: the scalar operator afterwards
    P.set_coeff_fields(None, None)
    assert np.array_equal(sb.axhelm(u, sb.HelmholtzCoeffs(0.7, 0.3), ctx, exact=True),
                          P.axhelm(u, 0.7, 0.3))
    ctx.close()


@pytest.mark.parametrize("case", CASES[:2], ids=lambda c: f"N{c[1]}")
@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_pcg_with_fields(cuda, refready, case, mode):
    dims, N, deform = case
    ctx = sb.Context.box(*dims, N, deform=deform)
    P = O.Problem(*dims, N, corners=O.box_corners(*dims, deform=deform), backend="ref")
    h1f, h2f = fields(P, 60 + N)
    P.set_coeff_fields(h1f, h2f)
    b = P.rhs_random_continuous(seed=5)
    ref = P.pcg(b, 1.0, 1.0, "jacobi", 1e-10, 2000)
    assert ref.converged
    co = sb.HelmholtzCoeffs(1.0, 1.0, h1_field=h1f, h2_field=h2f)
    x = np.zeros_like(b)
    r = sb.pcg(sb.HelmholtzOperator(ctx, co), b, x, sb.KrylovConfig(1e-10, 2000), mode=mode)
    # (FAST takes the reference-order path with fields: bitwise in both modes)
    assert r.iterations == ref.iterations
    assert np.array_equal(np.asarray(r.residual_history), ref.residual_history)
    assert np.array_equal(x, ref.x)
    # the batched call: every component as its single solve
    xs = [np.zeros_like(b) for _ in range(2)]
    rs = sb.pcg_multi(sb.HelmholtzOperator(ctx, co), [b, 0.5 * b], xs,
                      sb.KrylovConfig(1e-10, 2000), mode=mode)
    assert rs[0].iterations == ref.iterations and np.array_equal(xs[0], ref.x)
    ctx.close()


def test_fields_contract(cuda):
    ctx = sb.Context.box(2, 2, 2, 3)
    bad = np.ones(ctx.nodes - 1)
    with pytest.raises(sb.ContractViolation):
        sb.axhelm(np.zeros(ctx.nodes), sb.HelmholtzCoeffs(1.0, 0.0, h1_field=bad), ctx)
    ctx.close()
