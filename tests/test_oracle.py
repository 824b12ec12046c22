"""The CPU oracle (oracle/sbx_oracle.c) against the reference: golden vectors
from the unmodified reference (tests/golden/, made by make_golden.py) and,
where oracle/_ref was built, a live bitwise comparison."""
import hashlib

import numpy as np
import pytest

from oracle import oracle as O


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_rng_matches_libstdcxx(golden):
    # mt19937_64 + uniform_real_distribution: the seed-77 RHS hash pins it
    P = O.Problem(3, 3, 3, 4)
    b = P.rhs_random_continuous(77)
    assert sha(b) == golden["pcg_schwarz_b_sha"][0]


@pytest.mark.parametrize("N", range(1, 13))
def test_basis_bitwise(golden, N):
    P = O.Problem(1, 1, 1, N)
    assert np.array_equal(P.nodes, golden[f"basis_{N}_nodes"])
    assert np.array_equal(P.weights, golden[f"basis_{N}_weights"])
    assert np.array_equal(P.deriv, golden[f"basis_{N}_deriv"])


@pytest.mark.parametrize("tag", ["ax_a", "ax_b", "ax_c"])
def test_operators_bitwise(golden, tag):
    ex, ey, ez, N = golden[f"{tag}_dims"]
    cr = O.box_corners(ex, ey, ez, lengths=tuple(golden[f"{tag}_lengths"]),
                       deform=golden[f"{tag}_deform"][0])
    P = O.Problem(ex, ey, ez, N, lengths=tuple(golden[f"{tag}_lengths"]), corners=cr)
    u = golden[f"{tag}_u"]
    assert sha(np.concatenate([P.g1, P.g2, P.g3, P.g4, P.g5, P.g6, P.bm])) == \
        golden[f"{tag}_g_sha"][0]
    assert np.array_equal(P.axhelm(u, 0.9, 0.4), golden[f"{tag}_w"])
    assert np.array_equal(P.axhelm(u, 1.0, 0.0, flip=True), golden[f"{tag}_wflip"])
    assert np.array_equal(P.axhelm_diagonal(0.7, 1.3, assembled=True), golden[f"{tag}_diag"])
    f = u.copy()
    P.gs_sum_inplace(f)
    assert np.array_equal(f, golden[f"{tag}_gs"])
    assert np.array_equal(P.apply(u, 1.0, 1.0), golden[f"{tag}_apply"])
    assert P.dot_weighted(u, f) == golden[f"{tag}_dotw"][0]


@pytest.mark.parametrize("tag", ["gs_face", "gs_periodic_row", "gs_mixed", "gs_full_periodic",
                                 "gs_single_periodic"])
def test_gather_map_bitwise(golden, tag):
    ex, ey, ez, N, px, py, pz = golden[f"{tag}_dims"]
    P = O.Problem(ex, ey, ez, N, periodic=(bool(px), bool(py), bool(pz)))
    assert np.array_equal(P.group_offsets, golden[f"{tag}_offsets"])
    assert np.array_equal(P.group_nodes, golden[f"{tag}_nodes"])
    assert np.array_equal(P.gid, golden[f"{tag}_gid"])
    assert np.array_equal(P.mask, golden[f"{tag}_mask"])


def test_gather_known_answers():
    # test_mesh.cpp:61-80: shared face has 9 two-copy groups, 45 globals;
    # the centre vertex of a 2x2x2 box has multiplicity 8
    P = O.Problem(2, 1, 1, 2)
    sizes = np.diff(P.group_offsets)
    assert (sizes == 2).sum() == 9 and P.global_count == 45
    assert O.Problem(2, 2, 2, 1).mult.max() == 8
    # test_mesh.cpp:82-115 periodic row: 4*64 - 4*16 globals, mult 1 or 2
    Q = O.Problem(4, 1, 1, 3, periodic=(True, False, False))
    assert Q.global_count == 4 * 64 - 4 * 16
    assert set(np.unique(Q.mult)) <= {1, 2}


@pytest.mark.parametrize("tag", ["rcb_cube", "rcb_slab", "rcb_c1"])
def test_rcb_bitwise(golden, tag):
    ex, ey, ez = golden[f"{tag}_dims"]
    cr = O.box_corners(ex, ey, ez, lengths=tuple(golden[f"{tag}_lengths"]),
                       deform=golden[f"{tag}_deform"][0])
    P = O.Problem(ex, ey, ez, 1, lengths=tuple(golden[f"{tag}_lengths"]), corners=cr)
    for r in (2, 3, 4, 5, 8, 16):
        key = f"{tag}_{r}"
        if key in golden:
            assert np.array_equal(P.partition_rcb(r), golden[key])


PCG_FAST = ["pcg_schwarz", "pcg_helm4", "pcg_c1_manu"]
PCG_SLOW = ["pcg_c1_rand", "pcg_c1_rand12", "pcg_helm10"]


def _pcg_case(golden, tag):
    ex, ey, ez, N, h2, tol, deform, rnd = golden[f"{tag}_cfg"]
    ex, ey, ez, N = int(ex), int(ey), int(ez), int(N)
    cr = O.box_corners(ex, ey, ez, deform=deform)
    P = O.Problem(ex, ey, ez, N, corners=cr)
    b = P.rhs_random_continuous(77) if rnd else P.rhs_manufactured(h2)
    return P, b, h2, tol


@pytest.mark.parametrize("tag", PCG_FAST + PCG_SLOW)
def test_pcg_bitwise(golden, tag):
    P, b, h2, tol = _pcg_case(golden, tag)
    assert sha(b) == golden[f"{tag}_b_sha"][0]
    res = P.pcg(b, 1.0, h2, "jacobi", tol, 5000)
    assert res.iterations == golden[f"{tag}_iterations"][0]
    assert np.array_equal(res.residual_history, golden[f"{tag}_history"])
    assert sha(res.x) == golden[f"{tag}_x_sha"][0]
    assert res.rel_residual == golden[f"{tag}_rel"][0]
    assert res.rel_residual_precond == golden[f"{tag}_rel"][1]


def test_pcg_edge_cases():
    P = O.Problem(2, 2, 2, 3)
    z = np.zeros(P.nodes_count)
    r = P.pcg(z, max_iterations=10)
    assert r.converged and r.iterations == 0 and not r.x.any()
    b = P.rhs_random_continuous(5)
    r = P.pcg(b, tol=1e-14, max_iterations=1)
    assert not r.converged and r.iterations == 1 and r.status == 0
    bn = b.copy()
    bn[7] = np.nan
    r = P.pcg(bn)
    assert r.status in (5, 6)


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("cfg", [(3, 2, 2, 4, (True, False, False), 0.0),
                                 (4, 3, 2, 6, (False, True, False), 0.03),
                                 (2, 2, 2, 9, (False, False, False), 0.05)])
def test_port_vs_live_reference(cfg):
    ex, ey, ez, N, per, deform = cfg
    cr = O.box_corners(ex, ey, ez, deform=deform)
    P = O.Problem(ex, ey, ez, N, periodic=per, corners=cr)
    R = O.Problem(ex, ey, ez, N, periodic=per, corners=cr, backend="ref")
    for k in ["g1", "g2", "g3", "g4", "g5", "g6", "bm", "mask", "inv_mult", "gid",
              "group_offsets", "group_nodes", "mult"]:
        assert np.array_equal(getattr(P, k), getattr(R, k)), k
    u = O.fill_uniform(3, P.nodes_count)
    assert np.array_equal(P.apply(u, 0.5, 2.0), R.apply(u, 0.5, 2.0))
    b = P.rhs_random_continuous(11)
    pr, rr = P.pcg(b, 0.5, 2.0, tol=1e-10), R.pcg(b, 0.5, 2.0, tol=1e-10)
    assert pr.iterations == rr.iterations
    assert np.array_equal(pr.residual_history, rr.residual_history)
    assert np.array_equal(pr.x, rr.x)


def test_dense_oracle_matches_axhelm():
    # test_operators.cpp:115-144: axhelm vs the O(n^6) dense quadrature oracle
    for N in (1, 2, 3, 4):
        P = O.Problem(2, 1, 1, N, lengths=(1.4, 1.0, 0.8))
        u = O.fill_uniform(100 + N, P.nodes_count)
        w = P.axhelm(u, 0.9, 0.4)
        nn = P.nper
        for e in range(P.E):
            A = P.dense_helmholtz_element(e, 0.9, 0.4)
            np.testing.assert_allclose(w[e * nn:(e + 1) * nn], A @ u[e * nn:(e + 1) * nn],
                                       rtol=1e-11, atol=1e-11)
