"""TEST INFRASTRUCTURE ONLY -- ctypes front-end of the CPU oracle.

Two back-ends with the same Python surface:

* ``Port``  -- oracle/liboracle.so, the plain-C restatement (oracle/sbx_oracle.c)
  of the reference's hot path.  Always buildable (gcc), travels to the GPU box.
* ``Ref``   -- oracle/_ref/libsembox_ref.so, the UNMODIFIED reference sources
  (/root/reference/proj/src) compiled by oracle/Makefile plus ref_shim.cpp.
  Built here (where /root/reference exists); the built .so travels to the box.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may import
this module.  The product package (paper_2109_03592_b200/) never does.

Both back-ends build a ``Problem``: a box mesh (optionally with caller-given
deformed corners), the GLL basis, geometric factors, gather-scatter map and
Dirichlet mask -- everything ``HelmholtzOperator`` needs
(proj/include/sembox/operators.hpp:103-112).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsembox_ref.so")

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
_P = C.c_void_p


class OracleError(RuntimeError):
    def __init__(self, code, msg, iteration=-1):
        super().__init__(msg)
        self.code = code
        self.iteration = iteration


def build(ref: bool = True) -> None:
    """Compile the C restatement (and, if /root/reference exists, oracle/_ref)."""
    import subprocess

    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-C", HERE, "ref", "-j8"], check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


# ----------------------------------------------------------------- inputs --
def fill_uniform(seed: int, n: int, a: float = -1.0, b: float = 1.0) -> np.ndarray:
    """std::mt19937_64(seed) + uniform_real_distribution(a, b) (libstdc++)."""
    out = np.empty(n, dtype=np.float64)
    _port().or_fill_uniform(C.c_uint64(seed), C.c_int64(n), a, b, out)
    return out


def box_corners(ex, ey, ez, origin=(0.0, 0.0, 0.0), lengths=(1.0, 1.0, 1.0), deform=0.0):
    """Corners [E,8,3] of build_box_mesh (mesh.cpp:21-52), optionally with the
    conforming sin-bump deformation of the benchmark configs."""
    E = ex * ey * ez
    out = np.empty((E, 8, 3), dtype=np.float64)
    lib = _port()
    rc = lib.or_box_corners(ex, ey, ez, np.asarray(origin, np.float64),
                            np.asarray(lengths, np.float64), out.reshape(-1))
    if rc:
        raise OracleError(rc, "build_box_mesh: bad configuration")
    if deform != 0.0:
        lib.or_deform_corners(C.c_int64(E), deform, out.reshape(-1))
    return out


# ----------------------------------------------------------------- port ----
_PORT = None
_REF = None


def _port():
    global _PORT
    if _PORT is None:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        L = C.CDLL(PORT_SO)
        L.or_fill_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _dp]
        L.or_gll_basis.argtypes = [C.c_int, _dp, _dp, _dp]
        L.or_box_corners.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        L.or_deform_corners.argtypes = [C.c_int64, C.c_double, _dp]
        L.or_trilinear_point.argtypes = [_dp, C.c_int64, C.c_double, C.c_double, C.c_double, _dp]
        L.or_geometric_factors.restype = C.c_int64
        L.or_geometric_factors.argtypes = [C.c_int64, C.c_int, _dp, _dp, _dp] + [_dp] * 8
        L.or_gather_scatter.restype = C.c_int64
        L.or_gather_scatter.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, C.c_int,
                                        _i64p, _i64p, _i64p, _i32p, _dp]
        L.or_dirichlet_mask.argtypes = [C.c_int, C.c_int, C.c_int, _i32p, C.c_int, _dp]
        L.or_axhelm.argtypes = [C.c_int64, C.c_int] + [_dp] * 8 + [C.c_double, C.c_double,
                                                                   C.c_int, _dp, _dp]
        L.or_axhelm_diagonal.argtypes = [C.c_int64, C.c_int] + [_dp] * 8 + [
            C.c_double, C.c_double, _dp]
        L.or_gs_sum.argtypes = [C.c_int64, _i64p, _i64p, _dp]
        L.or_dot_weighted.restype = C.c_double
        L.or_dot_weighted.argtypes = [C.c_int64, C.c_int, _dp, _dp, C.c_void_p]
        L.or_pcg.restype = C.c_int
        L.or_pcg.argtypes = ([C.c_int64, C.c_int] + [_dp] * 11 + [C.c_int64, _i64p, _i64p,
                             C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_double, C.c_int,
                             _i64p, _dp, _dp, C.c_int64, _i64p])
        L.or_partition_rcb.argtypes = [C.c_int64, _dp, C.c_int, _i32p]
        L.or_dense_helmholtz_element.argtypes = [_dp, C.c_int64, C.c_int, _dp, _dp, _dp,
                                                 C.c_double, C.c_double, _dp]
        _PORT = L
    return _PORT


def _ref():
    global _REF
    if _REF is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(
                f"{REF_SO} missing: build it with `make -C oracle ref` where /root/reference exists")
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_set_workers.argtypes = [C.c_int]
        L.ref_workers.restype = C.c_int
        L.ref_problem_create.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _i32p, C.c_int,
                                         C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.ref_problem_destroy.argtypes = [_P]
        L.ref_problem_sizes.argtypes = [_P, _i64p]
        L.ref_copy_double.argtypes = [_P, C.c_int, _dp]
        L.ref_copy_int64.argtypes = [_P, C.c_int, _i64p]
        L.ref_copy_mult.argtypes = [_P, _i32p]
        L.ref_axhelm.argtypes = [_P, _dp, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_set_coeff_fields.argtypes = [_P, C.c_void_p, C.c_void_p]
        L.ref_axhelm_diagonal.argtypes = [_P, C.c_double, C.c_double, C.c_int, _dp]
        L.ref_gs_sum.argtypes = [_P, _dp]
        L.ref_apply.argtypes = [_P, C.c_double, C.c_double, C.c_int, _dp, _dp]
        L.ref_dot_weighted.restype = C.c_double
        L.ref_dot_weighted.argtypes = [_P, _dp, _dp]
        L.ref_pcg.argtypes = [_P, C.c_double, C.c_double, C.c_int, _dp, _dp, C.c_double,
                              C.c_int, _i64p, _dp, _dp, C.c_int64, _i64p]
        L.ref_partition_rcb.argtypes = [_P, C.c_int, _i32p]
        L.ref_pressure_setup.argtypes = [_P]
        L.ref_pressure_copy.argtypes = [_P, C.c_int, _dp]
        L.ref_gradient_from_pressure.argtypes = [_P, _dp, _dp, _dp, _dp]
        L.ref_divergence_to_pressure.argtypes = [_P, _dp, _dp, _dp, _dp]
        L.ref_pressure_apply.argtypes = [_P, _dp, _dp]
        L.ref_pressure_pcg.argtypes = [_P, C.c_int, _dp, _dp, C.c_double, C.c_int, _i64p, _dp,
                                       _dp, C.c_int64, _i64p]
        L.ref_projection_reset.argtypes = [_P, C.c_int]
        L.ref_projection_size.argtypes = [_P]
        L.ref_projection_guess.argtypes = [_P, _dp, _dp, C.c_void_p]
        L.ref_projection_append.argtypes = [_P, _dp]
        L.ref_advect.argtypes = [_P] + [_dp] * 9
        L.ref_bench_prepare.argtypes = [_P, C.c_double, C.c_double, _dp]
        L.ref_bench_solve.argtypes = [_P, C.c_int, _i64p, _dp]
        L.ref_dense_helmholtz_element.argtypes = [_P, C.c_int, C.c_double, C.c_double, _dp]
        L.ref_trilinear_point.argtypes = [_P, C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        L.ref_fill_uniform.argtypes = [C.c_uint64, C.c_int64, C.c_double, C.c_double, _dp]
        _REF = L
    return _REF


@dataclass
class PcgOut:
    iterations: int
    converged: bool
    rel_residual: float
    rel_residual_precond: float
    residual_history: np.ndarray
    x: np.ndarray
    status: int = 0
    error_iteration: int = -1


@dataclass
class Problem:
    """Mesh + basis + geometry + gs map + mask for a (possibly deformed) box."""

    ex: int
    ey: int
    ez: int
    degree: int
    periodic: tuple = (False, False, False)
    origin: tuple = (0.0, 0.0, 0.0)
    lengths: tuple = (1.0, 1.0, 1.0)
    corners: np.ndarray | None = None
    backend: str = "port"  # "port" | "ref"
    with_gradients: bool = False  # ref backend: GeometricFactors with drdx (advect)
    # filled in
    E: int = field(init=False)
    n: int = field(init=False)

    def __post_init__(self):
        self.E = self.ex * self.ey * self.ez
        self.n = self.degree + 1
        self.nper = self.n ** 3
        self.nodes_count = self.E * self.nper
        per = np.asarray([1 if p else 0 for p in self.periodic], np.int32)
        self._per = per
        if self.corners is None:
            self.corners = box_corners(self.ex, self.ey, self.ez, self.origin, self.lengths)
        self.corners = np.ascontiguousarray(self.corners, np.float64)
        if self.backend == "ref":
            self._build_ref()
        else:
            self._build_port()

    # -- construction ---------------------------------------------------
    def _build_port(self):
        L = _port()
        n, E = self.n, self.E
        self.nodes = np.empty(n)
        self.weights = np.empty(n)
        self.deriv = np.empty(n * n)
        rc = L.or_gll_basis(self.degree, self.nodes, self.weights, self.deriv)
        if rc:
            raise OracleError(rc, "build_gll_basis: degree out of range")
        N = self.nodes_count
        g = [np.empty(N) for _ in range(8)]
        bad = L.or_geometric_factors(E, n, self.nodes, self.weights, self.corners.reshape(-1),
                                     *g)
        if bad >= 0:
            raise OracleError(4, f"build_geometric_factors: nonpositive Jacobian in element {bad}")
        self.g1, self.g2, self.g3, self.g4, self.g5, self.g6, self.bm, self.jac = g
        self.gid = np.empty(N, np.int64)
        offs = np.empty(N + 1, np.int64)
        self.group_nodes = np.empty(N, np.int64)
        self.mult = np.empty(N, np.int32)
        self.inv_mult = np.empty(N)
        G = L.or_gather_scatter(self.ex, self.ey, self.ez, self._per, self.degree, self.gid,
                                offs, self.group_nodes, self.mult, self.inv_mult)
        self.global_count = int(G)
        self.group_offsets = offs[: G + 1].copy()
        self.mask = np.empty(N)
        L.or_dirichlet_mask(self.ex, self.ey, self.ez, self._per, self.degree, self.mask)

    def _build_ref(self):
        L = _ref()
        h = C.c_void_p()
        rc = L.ref_problem_create(self.ex, self.ey, self.ez, np.asarray(self.origin, np.float64),
                                  np.asarray(self.lengths, np.float64), self._per, self.degree,
                                  self.corners.ctypes.data_as(C.c_void_p),
                                  int(self.with_gradients), C.byref(h))
        if rc:
            raise OracleError(rc, L.ref_last_error().decode())
        self._h = h
        sizes = np.empty(4, np.int64)
        L.ref_problem_sizes(h, sizes)
        self.global_count = int(sizes[3])
        # the reference's arrays are copied out on first use (__getattr__):
        # at the benchmark size (64^3, N=7) each one is a 1 GB host array

    # reference-owned arrays fetched lazily: name -> (kind, which, count)
    _REF_ARRAYS = {"nodes": ("d", 0, "n"), "weights": ("d", 1, "n"), "deriv": ("d", 2, "nn"),
                   "g1": ("d", 3, "N"), "g2": ("d", 4, "N"), "g3": ("d", 5, "N"),
                   "g4": ("d", 6, "N"), "g5": ("d", 7, "N"), "g6": ("d", 8, "N"),
                   "bm": ("d", 9, "N"), "jac": ("d", 10, "N"), "mask": ("d", 11, "N"),
                   "inv_mult": ("d", 12, "N"), "gid": ("i", 0, "N"),
                   "group_offsets": ("i", 1, "G1"), "group_nodes": ("i", 2, "N"),
                   "mult": ("m", 0, "N")}

    def __getattr__(self, name):
        spec = Problem._REF_ARRAYS.get(name)
        d = self.__dict__
        if spec is None or d.get("backend") != "ref" or d.get("_h") is None:
            raise AttributeError(name)
        kind, which, cnt = spec
        count = {"n": d["n"], "nn": d["n"] ** 2, "N": d["nodes_count"],
                 "G1": d["global_count"] + 1}[cnt]
        L = _ref()
        if kind == "d":
            a = np.empty(count)
            L.ref_copy_double(d["_h"], which, a)
        elif kind == "i":
            a = np.empty(count, np.int64)
            L.ref_copy_int64(d["_h"], which, a)
        else:
            a = np.empty(count, np.int32)
            L.ref_copy_mult(d["_h"], a)
        setattr(self, name, a)
        return a

    def drop(self, *names):
        """Release lazily fetched reference arrays (memory at large sizes)."""
        for nm in names:
            self.__dict__.pop(nm, None)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _REF is not None:
            _REF.ref_problem_destroy(h)
            self._h = None

    # -- operators --------------------------------------------------------
    def _gargs(self):
        return (self.deriv, self.g1, self.g2, self.g3, self.g4, self.g5, self.g6, self.bm)

    def set_coeff_fields(self, h1f=None, h2f=None):
        """HelmholtzCoeffs::h1_field / h2_field (operators.hpp:42-43) for every
        later operator and pcg of this (reference-backed) problem; None: the
        scalar."""
        assert self.backend == "ref", "per-node coefficients: reference backend only"
        self._cf = [None if f is None else np.ascontiguousarray(f, np.float64)
                    for f in (h1f, h2f)]
        _ref().ref_set_coeff_fields(self._h, *[None if f is None else f.ctypes.data
                                               for f in self._cf])

    def axhelm(self, u, h1=1.0, h2=0.0, flip=False):
        u = np.ascontiguousarray(u, np.float64)
        out = np.empty(self.nodes_count)
        if self.backend == "ref":
            rc = _ref().ref_axhelm(self._h, u, h1, h2, int(flip), out)
            if rc:
                raise OracleError(rc, _ref().ref_last_error().decode())
        else:
            _port().or_axhelm(self.E, self.n, *self._gargs(), h1, h2, int(flip), u, out)
        return out

    def axhelm_diagonal(self, h1=1.0, h2=0.0, assembled=False):
        out = np.empty(self.nodes_count)
        if self.backend == "ref":
            _ref().ref_axhelm_diagonal(self._h, h1, h2, int(assembled), out)
        else:
            _port().or_axhelm_diagonal(self.E, self.n, *self._gargs(), h1, h2, out)
            if assembled:
                self.gs_sum_inplace(out)
        return out

    def gs_sum_inplace(self, f):
        assert f.dtype == np.float64 and f.flags.c_contiguous
        if self.backend == "ref":
            _ref().ref_gs_sum(self._h, f)
        else:
            _port().or_gs_sum(self.global_count, self.group_offsets, self.group_nodes, f)
        return f

    def apply(self, x, h1=1.0, h2=0.0, use_mask=True):
        """HelmholtzOperator::apply (operators.cpp:530-534)."""
        x = np.ascontiguousarray(x, np.float64)
        if self.backend == "ref":
            out = np.empty(self.nodes_count)
            _ref().ref_apply(self._h, h1, h2, int(use_mask), x, out)
            return out
        out = self.axhelm(x, h1, h2)
        self.gs_sum_inplace(out)
        if use_mask:
            out *= self.mask
        return out

    def dot_weighted(self, a, b):
        a = np.ascontiguousarray(a, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        if self.backend == "ref":
            return _ref().ref_dot_weighted(self._h, a, b)
        return _port().or_dot_weighted(self.E, self.nper, a, b,
                                       self.inv_mult.ctypes.data_as(C.c_void_p))

    def pcg(self, b, h1=1.0, h2=0.0, precond="jacobi", tol=1e-8, max_iterations=500,
            x0=None, hist_cap=None):
        pc = {"none": 0, None: 0, "jacobi": 1}[precond]
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.nodes_count) if x0 is None else np.array(x0, np.float64)
        info = np.zeros(3, np.int64)
        res = np.zeros(2)
        cap = (max_iterations + 1) if hist_cap is None else hist_cap
        hist = np.zeros(cap)
        hlen = np.zeros(1, np.int64)
        if self.backend == "ref":
            rc = _ref().ref_pcg(self._h, h1, h2, pc, b, x, tol, max_iterations, info, res, hist,
                                cap, hlen)
        else:
            diag = self.axhelm_diagonal(h1, h2, assembled=True)
            rc = _port().or_pcg(self.E, self.n, *self._gargs(), self.mask, self.inv_mult, diag,
                                self.global_count, self.group_offsets, self.group_nodes, h1,
                                h2, pc, b, x, tol, max_iterations, info, res, hist, cap, hlen)
        return PcgOut(int(info[0]), bool(info[1]), float(res[0]), float(res[1]),
                      hist[: min(int(hlen[0]), cap)].copy(), x, int(rc), int(info[2]))

    # -- consistent-Poisson pressure path (reference backend only) ---------
    # stepper.cpp:59-84 setup, operators.cpp:327-410, stepper.cpp:240-348
    def pressure_setup(self):
        assert self.backend == "ref"
        rc = _ref().ref_pressure_setup(self._h)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        self.m = self.degree - 1
        self.pnodes_count = self.E * self.m ** 3

    def pressure_array(self, which):
        """0 GL nodes, 1 GL weights, 2 interp_v2p, 3 wdetj, 4 drdx, 5 inv_bdiag,
        6 the Jacobi diagonal (pressure_operator_diagonal)."""
        m, n = self.m, self.n
        count = [m, m, m * n, self.pnodes_count, 9 * self.pnodes_count, self.nodes_count,
                 self.pnodes_count][which]
        out = np.empty(count)
        _ref().ref_pressure_copy(self._h, which, out)
        return out

    def gradient_from_pressure(self, p):
        g = [np.empty(self.nodes_count) for _ in range(3)]
        rc = _ref().ref_gradient_from_pressure(self._h, np.ascontiguousarray(p, np.float64), *g)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return g

    def divergence_to_pressure(self, ux, uy, uz):
        out = np.empty(self.pnodes_count)
        rc = _ref().ref_divergence_to_pressure(self._h, *[np.ascontiguousarray(u, np.float64)
                                                          for u in (ux, uy, uz)], out)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return out

    def pressure_apply(self, p):
        out = np.empty(self.pnodes_count)
        rc = _ref().ref_pressure_apply(self._h, np.ascontiguousarray(p, np.float64), out)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return out

    def pressure_pcg(self, b, precond="jacobi", tol=1e-6, max_iterations=500, x0=None):
        pc = {"none": 0, None: 0, "jacobi": 1}[precond]
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.pnodes_count) if x0 is None else np.array(x0, np.float64)
        info = np.zeros(3, np.int64)
        res = np.zeros(2)
        cap = max_iterations + 1
        hist = np.zeros(cap)
        hlen = np.zeros(1, np.int64)
        rc = _ref().ref_pressure_pcg(self._h, pc, b, x, tol, max_iterations, info, res, hist,
                                     cap, hlen)
        return PcgOut(int(info[0]), bool(info[1]), float(res[0]), float(res[1]),
                      hist[: min(int(hlen[0]), cap)].copy(), x, int(rc), int(info[2]))

    def projection_reset(self, depth):
        _ref().ref_projection_reset(self._h, depth)

    def projection_size(self):
        return _ref().ref_projection_size(self._h)

    def projection_guess(self, b, deflated=False):
        g = np.empty(self.pnodes_count)
        d = np.empty(self.pnodes_count) if deflated else None
        rc = _ref().ref_projection_guess(self._h, np.ascontiguousarray(b, np.float64), g,
                                         None if d is None else d.ctypes.data_as(C.c_void_p))
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return (g, d) if deflated else g

    def projection_append(self, x):
        rc = _ref().ref_projection_append(self._h, np.ascontiguousarray(x, np.float64))
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())

    def advect(self, u, c):
        out = [np.empty(self.nodes_count) for _ in range(3)]
        rc = _ref().ref_advect(self._h, *[np.ascontiguousarray(v, np.float64) for v in u],
                               *[np.ascontiguousarray(v, np.float64) for v in c], *out)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return out

    def pressure_rhs(self, seed=5):
        """A pressure right-hand side as solve_pressure_update forms it
        (stepper.cpp:311-324): the divergence of a random continuous, masked
        velocity field, mean removed."""
        u = []
        for d in range(3):
            f = fill_uniform(seed + d, self.nodes_count)
            self.gs_sum_inplace(f)
            f *= self.inv_mult * self.mask
            u.append(f)
        rhs = self.divergence_to_pressure(*u)
        rhs -= rhs.sum() / rhs.size
        return rhs

    # -- benchmark session (reference backend only) ------------------------
    def bench_prepare(self, b, h1=1.0, h2=0.0):
        """Untimed setup of a timed reference solve: the assembled Jacobi
        diagonal and the right-hand side stay inside the reference problem."""
        assert self.backend == "ref"
        rc = _ref().ref_bench_prepare(self._h, h1, h2, np.ascontiguousarray(b, np.float64))
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())

    def bench_solve(self, iters):
        """x = 0, then the reference pcg for exactly `iters` iterations."""
        info = np.zeros(3, np.int64)
        res = np.zeros(2)
        rc = _ref().ref_bench_solve(self._h, iters, info, res)
        if rc:
            raise OracleError(rc, _ref().ref_last_error().decode())
        return int(info[0])

    def partition_rcb(self, ranks):
        out = np.empty(self.E, np.int32)
        if self.backend == "ref":
            rc = _ref().ref_partition_rcb(self._h, ranks, out)
        else:
            rc = _port().or_partition_rcb(self.E, self.corners.reshape(-1), ranks, out)
        if rc:
            raise OracleError(rc, "partition_rcb: bad rank count")
        return out

    def dense_helmholtz_element(self, elem, h1, h2):
        nn = self.nper
        out = np.empty(nn * nn)
        if self.backend == "ref":
            _ref().ref_dense_helmholtz_element(self._h, elem, h1, h2, out)
        else:
            _port().or_dense_helmholtz_element(self.corners.reshape(-1), elem, self.n,
                                               self.nodes, self.weights, self.deriv, h1, h2,
                                               out)
        return out.reshape(nn, nn)

    def node_coords(self):
        """Physical coordinates [N,3] of every local node (oracle.cpp:67-76)."""
        L = _port()
        out = np.empty((self.nodes_count, 3))
        x = np.empty(3)
        n = self.n
        a = 0
        flat = self.corners.reshape(-1)
        for e in range(self.E):
            for k in range(n):
                for j in range(n):
                    for i in range(n):
                        L.or_trilinear_point(flat, e, self.nodes[i], self.nodes[j],
                                             self.nodes[k], x)
                        out[a] = x
                        a += 1
        return out

    # -- canonical right-hand sides --------------------------------------
    def rhs_random_continuous(self, seed=77):
        """test_schwarz.cpp:30-38: U(-1,1) mt19937_64(seed) -> gs_sum -> *= inv_mult*mask."""
        f = fill_uniform(seed, self.nodes_count)
        self.gs_sum_inplace(f)
        f *= self.inv_mult * self.mask
        return f

    def rhs_manufactured(self, h2=0.0):
        """mask * gs(bm * (3 pi^2 + h2) sin(pi x) sin(pi y) sin(pi z)) at the node
        coordinates (acceptance.cpp:74-87)."""
        xyz = self.node_coords()
        pi = math.pi
        u = np.sin(pi * xyz[:, 0]) * np.sin(pi * xyz[:, 1]) * np.sin(pi * xyz[:, 2])
        f = u * (3.0 * pi * pi + h2) * self.bm
        self.gs_sum_inplace(f)
        f *= self.mask
        return np.ascontiguousarray(f)
