"""Device-side setup of box contexts (setup_dev.cu) against
the host builders, which tests/test_setup.py pins bitwise to the reference
(operators.cpp:123-178, 433-455; gather.cpp:10-98):

* geometric factors g1..g6 and bm built by the GPU: bitwise equal;
* mask and inv_mult from the node lattice: bitwise equal;
* gs_sum on the lattice (no CSR): bitwise equal to the CSR gather-scatter of
  a from_problem context on the same mesh, with and without the mask;
* a nonpositive Jacobian raises MeshError naming the same element;
* SBX_HOST_SETUP=1 (the host path) gives the same arrays."""
import os
import subprocess
import sys
import time

import numpy as np
import pytest

import paper_2109_03592_b200 as sb
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CASES = [((3, 2, 2), 5, (False, False, False), 0.05),
         ((4, 3, 2), 7, (False, False, False), 0.05),
         ((2, 3, 2), 4, (True, False, False), 0.03),
         ((2, 2, 3), 6, (False, True, True), 0.0),
         ((2, 2, 2), 9, (True, True, True), 0.02),
         ((3, 1, 2), 3, (False, False, False), 0.04),
         ((2, 2, 2), 1, (False, False, False), 0.05)]


def host_problem(dims, N, per, deform):
    mesh = sb.build_box_mesh(*dims, periodic=per, deform=deform)
    basis = sb.build_gll_basis(N)
    gf = sb.build_geometric_factors(mesh, basis)
    gmap = sb.build_gather_scatter(mesh, N)
    mask = sb.build_dirichlet_mask(mesh, N)
    return mesh, basis, gf, gmap, mask


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"N{c[1]}-{''.join('p' if p else 'n' for p in c[2])}")
def test_device_setup_bitwise(cuda, case):
    dims, N, per, deform = case
    mesh, basis, gf, gmap, mask = host_problem(dims, N, per, deform)
    ctx = sb.Context.box(*dims, N, periodic=per, deform=deform)
    assert ctx.global_count == gmap.global_count
    for which, ref in ((0, mask), (1, gmap.inv_mult), (2, gf.bm), (3, gf.g1), (4, gf.g2),
                       (5, gf.g3), (6, gf.g4), (7, gf.g5), (8, gf.g6)):
        got = ctx.array(which)
        assert np.array_equal(got, ref), which
    # gather-scatter on the lattice vs the CSR gather-scatter of the same mesh
    pctx = sb.Context.from_problem(gf, basis, gmap, mask)
    u = O.fill_uniform(40 + N, ctx.nodes)
    assert np.array_equal(sb.gs_sum(ctx, u), sb.gs_sum(pctx, u))
    P = O.Problem(*dims, N, periodic=per, corners=mesh.corners)
    g = u.copy()
    P.gs_sum_inplace(g)
    assert np.array_equal(sb.gs_sum(ctx, u), g)
    for use_mask in (True, False):
        a = np.empty_like(u)
        b = np.empty_like(u)
        sb.HelmholtzOperator(ctx, sb.HelmholtzCoeffs(0.5, 2.0), use_mask=use_mask,
                             exact=True).apply(u, a)
        sb.HelmholtzOperator(pctx, sb.HelmholtzCoeffs(0.5, 2.0), use_mask=use_mask,
                             exact=True).apply(u, b)
        assert np.array_equal(a, b)
        assert np.array_equal(a, P.apply(u, 0.5, 2.0, use_mask=use_mask))
    assert np.array_equal(sb.HelmholtzOperator(ctx).assembled_diagonal(),
                          P.axhelm_diagonal(1.0, 0.0, assembled=True))
    ctx.close()
    pctx.close()


def test_device_setup_mesh_error(cuda):
    dims, N, deform = (3, 3, 3), 3, 0.6  # folds elements: detJ <= 0 somewhere
    mesh = sb.build_box_mesh(*dims, deform=deform)
    with pytest.raises(sb.MeshError) as host_err:
        sb.build_geometric_factors(mesh, sb.build_gll_basis(N))
    with pytest.raises(sb.MeshError) as dev_err:
        sb.Context.box(*dims, N, deform=deform)
    assert str(host_err.value).split()[-1] == str(dev_err.value).split()[-1]


def test_host_setup_switch_matches(cuda):
    """SBX_HOST_SETUP=1 (host builders + CSR upload) and the device path give
    the same context arrays and the same FAST solve."""
    code = (
        "import numpy as np, paper_2109_03592_b200 as sb;"
        "c = sb.Context.box(5, 4, 3, 7, deform=0.05);"
        "a = np.concatenate([c.array(w) for w in range(9)]);"
        "np.save('gpurun_out/_setup_arrays.npy', a)")
    os.makedirs("gpurun_out", exist_ok=True)
    subprocess.run([sys.executable, "-c", code], check=True,
                   env=dict(os.environ, SBX_HOST_SETUP="1"), cwd=os.path.dirname(
                       os.path.dirname(os.path.abspath(__file__))))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    host = np.load(os.path.join(root, "gpurun_out", "_setup_arrays.npy"))
    c = sb.Context.box(5, 4, 3, 7, deform=0.05)
    dev = np.concatenate([c.array(w) for w in range(9)])
    assert np.array_equal(host, dev)
    c.close()


def test_device_setup_time_bench_mesh(cuda):
    """The bench mesh (64^3, N=7) sets up in well under the 9.6 s of the host
    path (round 1); recorded, bounded loosely."""
    t = time.perf_counter()
    c = sb.Context.box(64, 64, 64, 7, deform=0.05)
    dt = time.perf_counter() - t
    print(f"setup 64^3 N=7: {dt:.2f} s")
    assert c.nodes == 64 ** 3 * 512
    c.close()
    assert dt < 3.0


def test_problem_with_box_hint_runs_the_box_kernels(cuda):
    """sbx_problem_desc's structured-box hint (the reference's HexMesh): the
    reference-layout map / mask / geometry are verified on the device, then
    the context runs exactly the kernels of Context.box -- identical bits."""
    torch = cuda
    dims, N, deform = (5, 4, 3), 7, 0.05
    mesh, basis, gf, gmap, mask = host_problem(dims, N, (False,) * 3, deform)
    hinted = sb.Context.from_problem(gf, basis, gmap, mask, mesh=mesh)
    plain = sb.Context.from_problem(gf, basis, gmap, mask)
    box = sb.Context.box(*dims, N, deform=deform)
    assert hinted.features() == {"lattice_gs", "box_k2", "trilinear"}
    assert plain.features() == set()
    assert box.features() == {"lattice_gs", "box_k2", "trilinear"}
    P = O.Problem(*dims, N, corners=mesh.corners)
    b = torch.from_numpy(P.rhs_random_continuous(77)).cuda()
    xs = []
    for ctx in (hinted, box, plain):
        x = torch.zeros_like(b)
        r = sb.pcg(sb.HelmholtzOperator(ctx), b, x, sb.KrylovConfig(1e-9, 2000))
        xs.append((r.iterations, x))
    assert xs[0][0] == xs[1][0] == xs[2][0]
    assert torch.equal(xs[0][1], xs[1][1])
    assert float((xs[0][1] - xs[2][1]).norm() / xs[2][1].norm()) <= 1e-10


def test_box_hint_that_does_not_match_is_ignored(cuda):
    dims, N, deform = (3, 3, 2), 5, 0.05
    mesh, basis, gf, gmap, mask = host_problem(dims, N, (False,) * 3, deform)
    # geometry that is not the corners' trilinear metric: lattice gs, stored G
    g2 = sb.GeometricFactors(gf.elem_count, gf.n1d, gf.g1 * 1.5, gf.g2, gf.g3, gf.g4, gf.g5,
                             gf.g6, gf.bm, gf.jac)
    ctx = sb.Context.from_problem(g2, basis, gmap, mask, mesh=mesh)
    assert ctx.features() == {"lattice_gs", "box_k2"}
    # a mask that is not the box's Dirichlet mask: the general CSR path
    m2 = mask.copy()
    m2[7] = 1.0 - m2[7]
    ctx2 = sb.Context.from_problem(gf, basis, gmap, m2, mesh=mesh)
    assert ctx2.features() == set()
    u = O.fill_uniform(3, ctx2.nodes)
    P = O.Problem(*dims, N, corners=mesh.corners)
    want = P.axhelm(u, 1.0, 0.0)
    P.gs_sum_inplace(want)
    got = np.empty_like(u)
    sb.HelmholtzOperator(ctx2, use_mask=False, exact=True).apply(u, got)
    assert np.array_equal(got, want)
    # a mesh hint of the wrong shape: ignored
    mesh3 = sb.build_box_mesh(3, 2, 3, deform=deform)
    ctx3 = sb.Context.from_problem(gf, basis, gmap, mask, mesh=mesh3)
    assert ctx3.features() == set()
