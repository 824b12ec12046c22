"""Product host-side builders (libsbx.so, C++; no GPU needed) against the
oracle and the reference golden vectors: floating-point outputs bitwise,
integer outputs (gather map, partition) bit-exact."""
import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O


@pytest.mark.parametrize("N", range(1, 13))
def test_gll_basis_bitwise(golden, N):
    b = sb.build_gll_basis(N)
    assert np.array_equal(b.nodes, golden[f"basis_{N}_nodes"])
    assert np.array_equal(b.weights, golden[f"basis_{N}_weights"])
    assert np.array_equal(b.deriv, golden[f"basis_{N}_deriv"])


def test_basis_rejects_bad_degree():
    for bad in (0, 33, -1):
        with pytest.raises(sb.ConfigError):
            sb.build_gll_basis(bad)


@pytest.mark.parametrize("cfg", [(2, 1, 1, 3, (1.4, 1.0, 0.8), 0.0),
                                 (3, 2, 2, 5, (1.0, 1.0, 1.0), 0.05),
                                 (8, 8, 8, 7, (1.0, 1.0, 1.0), 0.05),
                                 (5, 3, 4, 2, (2.0, 0.7, 1.3), 0.02)])
def test_geometry_bitwise(cfg):
    ex, ey, ez, N, lengths, deform = cfg
    mesh = sb.build_box_mesh(ex, ey, ez, lengths=lengths, deform=deform)
    cr = O.box_corners(ex, ey, ez, lengths=lengths, deform=deform)
    assert np.array_equal(mesh.corners, cr)
    P = O.Problem(ex, ey, ez, N, lengths=lengths, corners=cr)
    gf = sb.build_geometric_factors(mesh, sb.build_gll_basis(N))
    for k in ["g1", "g2", "g3", "g4", "g5", "g6", "bm", "jac"]:
        assert np.array_equal(getattr(gf, k), getattr(P, k)), k


def test_nonpositive_jacobian_is_mesh_error():
    mesh = sb.build_box_mesh(1, 1, 1)
    mesh.corners[0, [0, 1]] = mesh.corners[0, [1, 0]]  # test_operators.cpp:109-113
    with pytest.raises(sb.MeshError):
        sb.build_geometric_factors(mesh, sb.build_gll_basis(2))


@pytest.mark.parametrize("tag", ["gs_face", "gs_periodic_row", "gs_mixed", "gs_full_periodic",
                                 "gs_single_periodic"])
def test_gather_map_bit_exact(golden, tag):
    ex, ey, ez, N, px, py, pz = golden[f"{tag}_dims"]
    mesh = sb.build_box_mesh(ex, ey, ez, periodic=(px, py, pz))
    m = sb.build_gather_scatter(mesh, N)
    assert np.array_equal(m.group_offsets, golden[f"{tag}_offsets"])
    assert np.array_equal(m.group_nodes, golden[f"{tag}_nodes"])
    assert np.array_equal(m.gid, golden[f"{tag}_gid"])
    assert np.array_equal(sb.build_dirichlet_mask(mesh, N), golden[f"{tag}_mask"])


@pytest.mark.parametrize("cfg", [(8, 8, 8, 7, (0, 0, 0)), (6, 5, 4, 3, (1, 0, 1)),
                                 (3, 1, 2, 5, (1, 1, 1)), (1, 2, 1, 4, (1, 0, 0))])
def test_gather_map_vs_oracle(cfg):
    ex, ey, ez, N, per = cfg
    mesh = sb.build_box_mesh(ex, ey, ez, periodic=per)
    m = sb.build_gather_scatter(mesh, N)
    P = O.Problem(ex, ey, ez, N, periodic=tuple(bool(p) for p in per))
    assert m.global_count == P.global_count
    for k in ["gid", "group_offsets", "group_nodes", "mult", "inv_mult"]:
        assert np.array_equal(getattr(m, k), getattr(P, k)), k


@pytest.mark.parametrize("tag", ["rcb_cube", "rcb_slab", "rcb_c1"])
def test_rcb_bit_exact(golden, tag):
    ex, ey, ez = golden[f"{tag}_dims"]
    mesh = sb.build_box_mesh(ex, ey, ez, lengths=tuple(golden[f"{tag}_lengths"]),
                             deform=golden[f"{tag}_deform"][0])
    for r in (2, 3, 4, 5, 8, 16):
        key = f"{tag}_{r}"
        if key in golden:
            assert np.array_equal(sb.partition_rcb(mesh, r), golden[key])
    with pytest.raises(sb.ConfigError):
        sb.partition_rcb(mesh, mesh.elem_count + 1)


def test_rcb_octants_and_balance():
    # test_mesh.cpp:203-241
    mesh = sb.build_box_mesh(4, 4, 4)
    p = sb.partition_rcb(mesh, 8)
    seen = set()
    for oz in range(2):
        for oy in range(2):
            for ox in range(2):
                inside = {int(p[e]) for e in range(64)
                          if tuple(c // 2 for c in mesh.elem_coords(e)) == (ox, oy, oz)}
                assert len(inside) == 1
                seen |= inside
    assert len(seen) == 8
    for ranks in (2, 3, 4, 8, 16, 64):
        cnt = np.bincount(sb.partition_rcb(mesh, ranks), minlength=ranks)
        assert cnt.min() >= 1 and cnt.max() <= 2 * cnt.min()


def test_pressure_basis_bitwise():
    """build_pressure_basis (basis.cpp:114-145): GL nodes, weights and the
    velocity-to-pressure interpolation, bitwise against the reference build."""
    import pytest

    from oracle import oracle as O

    if not O.ref_available():
        pytest.skip("oracle/_ref not built")
    for N in (3, 4, 5, 7, 8, 9, 12, 15):
        pb = sb.build_pressure_basis(N)
        P = O.Problem(2, 1, 1, N, backend="ref")
        P.pressure_setup()
        assert np.array_equal(pb.nodes, P.pressure_array(0)), N
        assert np.array_equal(pb.weights, P.pressure_array(1)), N
        assert np.array_equal(pb.interp_v2p, P.pressure_array(2)), N
