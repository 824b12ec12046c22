"""Generate tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run here, where /root/reference exists and `make -C oracle ref` has built
oracle/_ref/libsembox_ref.so:

    python tests/golden/make_golden.py

The fixtures pin the oracle restatement (tests/test_oracle.py) and, through
it, the CUDA path (tests/test_gpu_*.py).  Cases follow the reference's own
tests: test_basis.cpp, test_operators.cpp:115-171, test_mesh.cpp:61-250,
test_schwarz.cpp:156-193 (Jacobi branch), acceptance.cpp:68-119 and the
SURVEY.md section 8(c) C1 probe (8^3 deformed box, N=7, tol 1e-8).
"""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import oracle as O  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main():
    O.build(ref=True)
    assert O.ref_available(), "oracle/_ref missing"
    out = {}

    # basis (test_basis.cpp): N = 1..12
    for N in range(1, 13):
        R = O.Problem(1, 1, 1, N, backend="ref")
        out[f"basis_{N}_nodes"] = R.nodes
        out[f"basis_{N}_weights"] = R.weights
        out[f"basis_{N}_deriv"] = R.deriv

    # axhelm on a 2x1x1 box (test_operators.cpp:115-144), deformed 3x2x2 box
    for tag, (ex, ey, ez, N, lengths, deform) in {
        "ax_a": (2, 1, 1, 3, (1.4, 1.0, 0.8), 0.0),
        "ax_b": (3, 2, 2, 5, (1.0, 1.0, 1.0), 0.05),
        "ax_c": (2, 2, 2, 7, (1.0, 1.0, 1.0), 0.05),
    }.items():
        cr = O.box_corners(ex, ey, ez, lengths=lengths, deform=deform)
        R = O.Problem(ex, ey, ez, N, lengths=lengths, corners=cr, backend="ref")
        u = O.fill_uniform(100 + N, R.nodes_count)
        out[f"{tag}_dims"] = np.array([ex, ey, ez, N])
        out[f"{tag}_lengths"] = np.array(lengths)
        out[f"{tag}_deform"] = np.array([deform])
        out[f"{tag}_u"] = u
        out[f"{tag}_w"] = R.axhelm(u, 0.9, 0.4)
        out[f"{tag}_wflip"] = R.axhelm(u, 1.0, 0.0, flip=True)
        out[f"{tag}_diag"] = R.axhelm_diagonal(0.7, 1.3, assembled=True)
        f = u.copy()
        R.gs_sum_inplace(f)
        out[f"{tag}_gs"] = f
        out[f"{tag}_apply"] = R.apply(u, 1.0, 1.0)
        out[f"{tag}_dotw"] = np.array([R.dot_weighted(u, f)])
        out[f"{tag}_g_sha"] = np.array([sha(np.concatenate(
            [R.g1, R.g2, R.g3, R.g4, R.g5, R.g6, R.bm]))])

    # gather-scatter maps (test_mesh.cpp:61-201)
    for tag, (ex, ey, ez, N, per) in {
        "gs_face": (2, 1, 1, 2, (0, 0, 0)),
        "gs_periodic_row": (4, 1, 1, 3, (1, 0, 0)),
        "gs_mixed": (3, 3, 2, 4, (0, 1, 0)),
        "gs_full_periodic": (2, 3, 2, 3, (1, 1, 1)),
        "gs_single_periodic": (1, 1, 1, 2, (1, 1, 1)),
    }.items():
        R = O.Problem(ex, ey, ez, N, periodic=tuple(bool(p) for p in per), backend="ref")
        out[f"{tag}_dims"] = np.array([ex, ey, ez, N, *per])
        out[f"{tag}_offsets"] = R.group_offsets
        out[f"{tag}_nodes"] = R.group_nodes
        out[f"{tag}_gid"] = R.gid
        out[f"{tag}_mask"] = R.mask

    # RCB (test_mesh.cpp:203-250) incl. a deformed mesh
    for tag, (ex, ey, ez, lengths, deform) in {
        "rcb_cube": (4, 4, 4, (1, 1, 1), 0.0),
        "rcb_slab": (8, 2, 2, (8, 2, 2), 0.0),
        "rcb_c1": (8, 8, 8, (1, 1, 1), 0.05),
    }.items():
        cr = O.box_corners(ex, ey, ez, lengths=lengths, deform=deform)
        R = O.Problem(ex, ey, ez, 1, lengths=lengths, corners=cr, backend="ref")
        out[f"{tag}_dims"] = np.array([ex, ey, ez])
        out[f"{tag}_lengths"] = np.array(lengths, float)
        out[f"{tag}_deform"] = np.array([deform])
        for r in (2, 3, 4, 5, 8, 16):
            if r <= R.E:
                out[f"{tag}_{r}"] = R.partition_rcb(r)

    # PCG (krylov.cpp:7-91) cases
    pcg_cases = {
        # test_schwarz.cpp:156-193, Jacobi branch
        "pcg_schwarz": dict(ex=3, ey=3, ez=3, N=4, deform=0.0, rhs="random", h2=0.0, tol=1e-8),
        # SURVEY 8(c) C1 probe: manufactured RHS (i), deformed
        "pcg_c1_manu": dict(ex=8, ey=8, ez=8, N=7, deform=0.05, rhs="manufactured", h2=0.0,
                            tol=1e-8),
        # C1 with the seed-77 continuous masked RHS (ii), tol 1e-8 and 1e-12
        "pcg_c1_rand": dict(ex=8, ey=8, ez=8, N=7, deform=0.05, rhs="random", h2=0.0, tol=1e-8),
        "pcg_c1_rand12": dict(ex=8, ey=8, ez=8, N=7, deform=0.05, rhs="random", h2=0.0,
                              tol=1e-12),
        # acceptance.cpp:68-119 Helmholtz h1=h2=1 spectral convergence, N=4 and N=10
        "pcg_helm4": dict(ex=2, ey=2, ez=2, N=4, deform=0.0, rhs="manufactured", h2=1.0,
                          tol=1e-13),
        "pcg_helm10": dict(ex=2, ey=2, ez=2, N=10, deform=0.0, rhs="manufactured", h2=1.0,
                           tol=1e-13),
    }
    for tag, c in pcg_cases.items():
        cr = O.box_corners(c["ex"], c["ey"], c["ez"], deform=c["deform"])
        P = O.Problem(c["ex"], c["ey"], c["ez"], c["N"], corners=cr, backend="port")
        R = O.Problem(c["ex"], c["ey"], c["ez"], c["N"], corners=cr, backend="ref")
        b = P.rhs_random_continuous(77) if c["rhs"] == "random" else P.rhs_manufactured(c["h2"])
        res = R.pcg(b, 1.0, c["h2"], "jacobi", c["tol"], 5000)
        out[f"{tag}_cfg"] = np.array([c["ex"], c["ey"], c["ez"], c["N"], c["h2"], c["tol"],
                                      c["deform"], 1.0 if c["rhs"] == "random" else 0.0])
        out[f"{tag}_b_sha"] = np.array([sha(b)])
        out[f"{tag}_iterations"] = np.array([res.iterations])
        out[f"{tag}_rel"] = np.array([res.rel_residual, res.rel_residual_precond])
        out[f"{tag}_history"] = res.residual_history
        out[f"{tag}_x_sha"] = np.array([sha(res.x)])
        out[f"{tag}_x_norm"] = np.array([float(np.sqrt(np.dot(res.x, res.x)))])
        print(f"{tag}: {res.iterations} iterations, rel {res.rel_residual:.6e} "
              f"relp {res.rel_residual_precond:.6e}")

    np.savez_compressed(os.path.join(HERE, "sembox_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "sembox_golden.npz"),
          os.path.getsize(os.path.join(HERE, "sembox_golden.npz")), "bytes")


if __name__ == "__main__":
    main()
