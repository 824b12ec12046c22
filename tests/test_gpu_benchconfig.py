"""Parity at the benchmark's own configuration, against the UNMODIFIED
reference (oracle/_ref, the sembox sources compiled from /root/reference and
run on the GPU box's host cores): the 64^3-element N=7 deformed box
(a = 0.05) that bench.py times (BASELINE configs[2]/[3]).

* gather-scatter map (gid, group_offsets, group_nodes) and partition_rcb at
  P = 2/4/8: bit-exact (gather.cpp:10-83, mesh.cpp:168-226);
* HelmholtzOperator::apply on a continuous random field: FAST within 1e-12
  relative L2, EXACT bitwise (operators.cpp:530-534);
* the solver's own K1 (on-the-fly trilinear metric) against axhelm: 1e-12;
* a fixed 30-iteration pcg (tol 0): EXACT reproduces the residual history
  and x bit for bit; FAST's history agrees within 1e-10 relative
  (krylov.cpp:7-91).

Needs ~40 GB of host memory (the reference's own 64^3 data structures) and
the reference build in oracle/_ref; skipped otherwise."""
import os

import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

EX = EY = EZ = 64
N = 7
DEFORM = 0.05
ITERS = 30
AX_TOL = 1e-12
HIST_TOL = 1e-10


def _host_gb():
    try:
        import psutil

        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


@pytest.fixture(scope="module")
def ref():
    if not O.ref_available():
        pytest.skip("oracle/_ref (the reference build) is not present")
    if _host_gb() < 48:
        pytest.skip(f"needs ~48 GB free host memory, have {_host_gb():.0f}")
    O._ref().ref_set_workers(os.cpu_count() or 1)
    corners = O.box_corners(EX, EY, EZ, deform=DEFORM)
    P = O.Problem(EX, EY, EZ, N, corners=corners, backend="ref")
    yield P
    del P


@pytest.fixture(scope="module")
def ctx(cuda, ref):
    c = sb.Context.box(EX, EY, EZ, N, deform=DEFORM)
    yield c
    c.close()


def test_gather_scatter_map_bit_exact(ref):
    mesh = sb.build_box_mesh(EX, EY, EZ, deform=DEFORM)
    gm = sb.build_gather_scatter(mesh, N)
    assert gm.global_count == ref.global_count
    for name in ("group_offsets", "group_nodes", "gid"):
        ours = getattr(gm, name)
        theirs = getattr(ref, name)
        assert np.array_equal(ours, theirs), name
        ref.drop(name)
        del ours, theirs
    mult = ref.mult
    assert np.array_equal(gm.mult, mult)
    ref.drop("mult")


@pytest.mark.parametrize("ranks", [2, 4, 8])
def test_partition_rcb_bit_exact(ref, ranks):
    mesh = sb.build_box_mesh(EX, EY, EZ, deform=DEFORM)
    ours = sb.partition_rcb(mesh, ranks)
    theirs = ref.partition_rcb(ranks)
    assert np.array_equal(ours, theirs)
    assert np.bincount(ours, minlength=ranks).tolist() == [EX * EY * EZ // ranks] * ranks


def test_apply_and_k1(ctx, ref, cuda):
    torch = cuda
    u = ref.rhs_random_continuous(5)  # continuous, masked
    want = ref.apply(u, 1.0, 0.0)
    ud = torch.from_numpy(u).cuda()
    got = torch.empty_like(ud)
    sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0)).apply(ud, got)
    g = got.cpu().numpy()
    assert np.linalg.norm(g - want) / np.linalg.norm(want) <= AX_TOL
    sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0), exact=True).apply(ud, got)
    assert np.array_equal(got.cpu().numpy(), want)
    del want, g
    # the fused solver's element kernel (trilinear metric) vs the reference axhelm
    v = O.fill_uniform(9, ctx.nodes)
    for h2 in (0.0, 1.0):
        want = ref.axhelm(v, 1.0, h2)
        w = sb.debug_cg_k1(torch.from_numpy(v).cuda(), sb.HelmholtzCoeffs(1.0, h2), ctx)
        assert np.linalg.norm(w.cpu().numpy() - want) / np.linalg.norm(want) <= AX_TOL


def test_pcg_history_30_iterations(ctx, ref, cuda):
    torch = cuda
    b = ref.rhs_random_continuous(77)
    want = ref.pcg(b, 1.0, 0.0, "jacobi", 0.0, ITERS)
    assert want.iterations == ITERS and want.residual_history.size == ITERS + 1
    op = sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(1.0, 0.0))
    bd = torch.from_numpy(b).cuda()
    # FAST (the product path the bench times)
    x = torch.zeros_like(bd)
    r = sb.pcg(op, bd, x, sb.KrylovConfig(0.0, ITERS), mode="fast")
    h = np.asarray(r.residual_history)
    assert r.iterations == ITERS and h.size == ITERS + 1
    rel = np.abs(h - want.residual_history) / want.residual_history
    assert rel.max() <= HIST_TOL, rel.max()
    xf = x.cpu().numpy()
    assert np.linalg.norm(xf - want.x) / np.linalg.norm(want.x) <= HIST_TOL
    # EXACT (reference operation order): bit for bit
    x.zero_()
    r = sb.pcg(op, bd, x, sb.KrylovConfig(0.0, ITERS), mode="exact")
    assert np.array_equal(np.asarray(r.residual_history), want.residual_history)
    assert np.array_equal(x.cpu().numpy(), want.x)
