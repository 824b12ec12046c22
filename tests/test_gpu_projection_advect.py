"""SURVEY 8(f) row 4 on the device: the pressure solve's projection history
(ProjectionHistory, krylov.cpp:93-124, as solve_pressure_update uses it,
stepper.cpp:326-345) and advection (advect + grad_velocity,
operators.cpp:300-325, 412-431), against the unmodified reference
(oracle/_ref).  EXACT: bitwise; FAST: to round-off."""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def refready():
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")


def make(dims, N, deform, periodic=(False, False, False), grads=False):
    ctx = sb.Context.box(*dims, N, periodic=periodic, deform=deform)
    P = O.Problem(*dims, N, periodic=periodic, corners=O.box_corners(*dims, deform=deform),
                  backend="ref", with_gradients=grads)
    return ctx, P


@pytest.mark.parametrize("case", [((3, 2, 2), 3, 0.05, (False,) * 3),
                                  ((2, 3, 2), 5, 0.04, (False, True, False)),
                                  ((3, 2, 2), 7, 0.05, (False,) * 3),
                                  ((2, 2, 2), 10, 0.03, (True, True, True))],
                         ids=lambda c: f"N{c[1]}")
def test_advect_bitwise(cuda, refready, case):
    torch = cuda
    dims, N, deform, per = case
    ctx, P = make(dims, N, deform, per, grads=True)
    u = [O.fill_uniform(10 + q, P.nodes_count) for q in range(3)]
    c = [O.fill_uniform(20 + q, P.nodes_count) for q in range(3)]
    want = P.advect(u, c)
    got = sb.advect(u, c, ctx)
    for q in range(3):
        assert np.array_equal(got[q], want[q]), q
    # device tensors: same bits
    gd = sb.advect([torch.from_numpy(v).cuda() for v in u],
                   [torch.from_numpy(v).cuda() for v in c], ctx)
    for q in range(3):
        assert np.array_equal(gd[q].cpu().numpy(), want[q])
    ctx.close()


@pytest.mark.parametrize("exact", [True, False], ids=["exact", "fast"])
def test_projection_history(cuda, refready, exact):
    """A sequence of pressure solves with projected initial guesses, as
    solve_pressure_update runs them (depth 3, so the oldest pair is evicted)."""
    ctx, P = make((3, 3, 2), 5, 0.05)
    P.pressure_setup()
    P.projection_reset(3)
    E = sb.PressureOperator(ctx, exact=exact)
    H = sb.ProjectionHistory(ctx, 3, exact=exact)
    mode = "exact" if exact else "fast"
    for step in range(5):
        b = P.pressure_rhs(5 + 7 * step)
        gref, dref = P.projection_guess(b, deflated=True)
        g, d = H.project_guess(b, deflated_rhs=True)
        if exact:
            assert np.array_equal(g, gref) and np.array_equal(d, dref), step
        else:
            scale = max(np.linalg.norm(gref), 1e-300)
            assert np.linalg.norm(g - gref) <= 1e-11 * max(scale, np.linalg.norm(b)), step
        # solve from the projected guess, then append the solution
        ref = P.pressure_pcg(b, "jacobi", 1e-8, 3000, x0=gref)
        x = gref.copy()
        r = sb.pcg_pressure(E, b, x, sb.KrylovConfig(1e-8, 3000), mode=mode)
        if exact:
            assert r.iterations == ref.iterations and np.array_equal(x, ref.x)
        P.projection_append(ref.x)
        H.append(ref.x)
        assert H.size() == P.projection_size() == min(step + 1, 3)
    ctx.close()
