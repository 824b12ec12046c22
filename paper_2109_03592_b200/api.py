"""Python mirror of the reference's operator API on the PCG hot path.

Same names, argument meaning and error behaviour as sembox
(/root/reference/proj/include/sembox/*.hpp), backed by libsbx.so (C ABI,
include/sbx.h).  Setup builders return host numpy arrays in the reference
layout; fields passed to operators may be numpy arrays (host, staged through
the context) or CUDA float64 torch tensors (device, zero-copy).

    basis = build_gll_basis(7)                         # basis.hpp:46
    mesh  = build_box_mesh(8, 8, 8, deform=0.05)       # mesh.hpp:43
    gf    = build_geometric_factors(mesh, basis)       # operators.hpp:46
    gmap  = build_gather_scatter(mesh, 7)              # gather.hpp:33
    mask  = build_dirichlet_mask(mesh, 7)              # operators.hpp:90
    op    = HelmholtzOperator(gf, basis, gmap, mask, HelmholtzCoeffs(1.0, 0.0))
    res   = pcg(op, b, x, KrylovConfig(tolerance=1e-8), precond="jacobi")
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

lib = L.lib


# ------------------------------------------------------------------ errors --
class SemboxError(RuntimeError):
    pass


class ConfigError(SemboxError):
    """errors.hpp:10-13"""


class ContractViolation(SemboxError):
    """errors.hpp:16-19"""


class MeshError(SemboxError):
    """errors.hpp:22-25"""


class SolverError(SemboxError):
    """errors.hpp:28-33: carries the failing iteration."""

    def __init__(self, what, iteration):
        super().__init__(what)
        self.iteration = iteration


class CudaError(SemboxError):
    pass


def _check(rc, iteration=-1):
    if rc == 0:
        return
    msg = lib.sbx_last_error().decode(errors="replace")
    if rc == 2:
        raise ConfigError(msg)
    if rc == 3:
        raise ContractViolation(msg)
    if rc == 4:
        raise MeshError(msg)
    if rc in (5, 6):
        raise SolverError(msg, iteration)
    if rc == 1:
        raise ValueError(msg)
    if rc == 8:
        raise SemboxError("communicator: " + msg)
    raise CudaError(f"status {rc}: {msg}")


def _ptr(a):
    """Raw pointer of a numpy array or a torch tensor (host or device)."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if not a.flags.c_contiguous:
            raise ContractViolation("field must be C-contiguous")
        return a.ctypes.data
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ContractViolation("field must be contiguous")
        return a.data_ptr()
    raise TypeError(f"unsupported field type {type(a)}")


def _f64(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float64)
    if hasattr(a, "dtype"):
        import torch

        if a.dtype != torch.float64:
            raise ContractViolation("fields are float64")
        return a.contiguous()
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ basis --
@dataclass
class SpectralBasis:
    """basis.hpp:11-21"""

    order: int
    nodes: np.ndarray
    weights: np.ndarray
    deriv: np.ndarray  # (N+1)^2 row-major, deriv[i*n+j] = l_j'(x_i)

    def n(self):
        return self.order + 1

    def d(self, i, j):
        return self.deriv[i * self.n() + j]


def build_gll_basis(degree: int) -> SpectralBasis:
    """basis.hpp:46 / basis.cpp:60-95"""
    n = degree + 1
    nodes = np.zeros(max(n, 1))
    weights = np.zeros(max(n, 1))
    deriv = np.zeros(max(n * n, 1))
    _check(lib.sbx_gll_basis(degree, nodes.ctypes.data, weights.ctypes.data, deriv.ctypes.data))
    return SpectralBasis(degree, nodes, weights, deriv)


# ------------------------------------------------------------------- mesh --
@dataclass
class HexMesh:
    """mesh.hpp:14-37 (structured box; corners [E,8,3])"""

    ex: int
    ey: int
    ez: int
    origin: tuple
    lengths: tuple
    periodic: tuple
    corners: np.ndarray

    @property
    def elem_count(self):
        return self.ex * self.ey * self.ez

    def structured(self):
        return self.ex > 0

    def elem_coords(self, e):
        return (e % self.ex, (e // self.ex) % self.ey, e // (self.ex * self.ey))


def build_box_mesh(ex, ey, ez, origin=(0.0, 0.0, 0.0), lengths=(1.0, 1.0, 1.0),
                   periodic=(False, False, False), deform=0.0) -> HexMesh:
    """mesh.hpp:43-45 / mesh.cpp:21-75; deform = amplitude of the conforming
    sin-bump perturbation used by the benchmark meshes."""
    if ex < 1 or ey < 1 or ez < 1:
        raise ConfigError("build_box_mesh: element counts must be >= 1")
    corners = np.empty((ex * ey * ez, 8, 3))
    o = (C.c_double * 3)(*origin)
    ln = (C.c_double * 3)(*lengths)
    _check(lib.sbx_box_corners(ex, ey, ez, C.addressof(o), C.addressof(ln), corners.ctypes.data))
    if deform:
        _check(lib.sbx_deform_corners(corners.shape[0], float(deform), corners.ctypes.data))
    return HexMesh(ex, ey, ez, tuple(origin), tuple(lengths), tuple(bool(p) for p in periodic),
                   corners)


def partition_rcb(mesh: HexMesh, ranks: int) -> np.ndarray:
    """mesh.hpp:57 / mesh.cpp:168-226: rank_of[E] (int32)."""
    out = np.empty(mesh.elem_count, np.int32)
    _check(lib.sbx_partition_rcb(mesh.elem_count, mesh.corners.ctypes.data, ranks,
                                 out.ctypes.data))
    return out


# ------------------------------------------------------------- geometry ----
@dataclass
class GeometricFactors:
    """operators.hpp:18-26 (SoA, E*n^3 each)"""

    elem_count: int
    n1d: int
    g1: np.ndarray
    g2: np.ndarray
    g3: np.ndarray
    g4: np.ndarray
    g5: np.ndarray
    g6: np.ndarray
    bm: np.ndarray
    jac: np.ndarray


def build_geometric_factors(mesh: HexMesh, basis: SpectralBasis, with_gradients=False):
    """operators.hpp:46-48 / operators.cpp:123-178 (gradients are not on the
    PCG path and are not produced)."""
    n = basis.n()
    N = mesh.elem_count * n ** 3
    arr = [np.empty(N) for _ in range(8)]
    bad = C.c_int64(-1)
    _check(lib.sbx_geometric_factors(mesh.elem_count, basis.order, mesh.corners.ctypes.data,
                                     *[a.ctypes.data for a in arr], C.byref(bad)))
    return GeometricFactors(mesh.elem_count, n, *arr)


@dataclass
class GatherScatterMap:
    """gather.hpp:14-29"""

    elem_count: int
    n1d: int
    global_count: int
    gid: np.ndarray
    mult: np.ndarray
    inv_mult: np.ndarray
    group_offsets: np.ndarray
    group_nodes: np.ndarray

    def node_count(self):
        return self.gid.shape[0]


def build_gather_scatter(mesh: HexMesh, degree: int) -> GatherScatterMap:
    """gather.hpp:33 / gather.cpp:10-83 (bit-exact)."""
    if not mesh.structured():
        raise ContractViolation("build_gather_scatter: requires a structured mesh")
    if degree < 1:
        raise ContractViolation("build_gather_scatter: degree must be >= 1")
    n = degree + 1
    N = mesh.elem_count * n ** 3
    gid = np.empty(N, np.int64)
    offs = np.empty(N + 1, np.int64)
    nodes = np.empty(N, np.int64)
    mult = np.empty(N, np.int32)
    inv = np.empty(N)
    G = C.c_int64(0)
    per = (C.c_int * 3)(*[int(p) for p in mesh.periodic])
    _check(lib.sbx_gather_scatter(mesh.ex, mesh.ey, mesh.ez, C.addressof(per), degree,
                                  gid.ctypes.data, offs.ctypes.data, nodes.ctypes.data,
                                  mult.ctypes.data, inv.ctypes.data, C.byref(G)))
    return GatherScatterMap(mesh.elem_count, n, G.value, gid, mult, inv,
                            offs[: G.value + 1].copy(), nodes)


def build_dirichlet_mask(mesh: HexMesh, degree: int) -> np.ndarray:
    """operators.hpp:90 / operators.cpp:433-455"""
    if not mesh.structured():
        raise ContractViolation("build_dirichlet_mask: requires a structured mesh")
    n = degree + 1
    out = np.empty(mesh.elem_count * n ** 3)
    per = (C.c_int * 3)(*[int(p) for p in mesh.periodic])
    _check(lib.sbx_dirichlet_mask(mesh.ex, mesh.ey, mesh.ez, C.addressof(per), degree,
                                  out.ctypes.data))
    return out


# --------------------------------------------------------------- operator --
@dataclass
class HelmholtzCoeffs:
    """operators.hpp:39-44: scalar h1, h2, or per-node fields h1_field /
    h2_field (E*n^3 arrays, host or device; they replace the scalar at each
    node, operators.cpp:242, 258, 292-293)."""

    h1: float = 1.0
    h2: float = 0.0
    h1_field: Optional[object] = None
    h2_field: Optional[object] = None


@contextlib.contextmanager
def _coeff_fields(ctx, coeffs: HelmholtzCoeffs):
    """Per-node coefficients on the context for the duration of one call
    (sbx_ctx_set_coeff_fields)."""
    f1, f2 = coeffs.h1_field, coeffs.h2_field
    if f1 is None and f2 is None:
        yield
        return
    f1 = None if f1 is None else _f64(f1)
    f2 = None if f2 is None else _f64(f2)
    ctx._shape_check(*[f for f in (f1, f2) if f is not None])
    _check(lib.sbx_ctx_set_coeff_fields(ctx.handle, _ptr(f1) if f1 is not None else None,
                                        _ptr(f2) if f2 is not None else None))
    try:
        yield
    finally:
        lib.sbx_ctx_set_coeff_fields(ctx.handle, None, None)


@dataclass
class KrylovConfig:
    """krylov.hpp:18-22"""

    tolerance: float = 1e-8
    max_iterations: int = 500
    projection_depth: int = 0


@dataclass
class PcgResult:
    """krylov.hpp:24-30"""

    iterations: int = 0
    rel_residual: float = 0.0
    rel_residual_precond: float = 0.0
    converged: bool = False
    residual_history: list = field(default_factory=list)


class Context:
    """Device-resident operator data (one sbx_ctx).  Owns everything the
    HelmholtzOperator points at (operators.hpp:103-108)."""

    def __init__(self, handle, device=0):
        self._h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle
        self.device = device
        E, n, N, G, nbytes = C.c_int64(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(lib.sbx_ctx_info(self._h, C.byref(E), C.byref(n), C.byref(N), C.byref(G),
                                C.byref(nbytes)))
        self.elem_count, self.n1d, self.nodes = E.value, n.value, N.value
        self.global_count, self.device_bytes = G.value, nbytes.value

    @classmethod
    def from_problem(cls, gf: GeometricFactors, basis: SpectralBasis, gmap: GatherScatterMap,
                     mask: Optional[np.ndarray], device: int = 0, mesh: "HexMesh" = None):
        """HelmholtzOperator's inputs as the reference builds them.  `mesh`
        (optional) is the structured-box hint of sbx_problem_desc: the
        context verifies the map/mask/geometry against it on the device and
        then runs the lattice gather-scatter and the trilinear-metric K1."""
        if gf.n1d != basis.n() or gmap.n1d != basis.n() or gf.elem_count != gmap.elem_count:
            raise ContractViolation("HelmholtzOperator: grid/shape mismatch")
        keep = [np.ascontiguousarray(a, np.float64) for a in
                (basis.deriv, gf.g1, gf.g2, gf.g3, gf.g4, gf.g5, gf.g6, gf.bm)]
        offs = np.ascontiguousarray(gmap.group_offsets, np.int64)
        nodes = np.ascontiguousarray(gmap.group_nodes, np.int64)
        m = None if mask is None else np.ascontiguousarray(mask, np.float64)
        d = L.ProblemDesc()
        d.elem_count = gf.elem_count
        d.degree = basis.order
        d.deriv = keep[0].ctypes.data
        for q in range(6):
            d.g[q] = keep[1 + q].ctypes.data
        d.bm = keep[7].ctypes.data
        d.mask = None if m is None else m.ctypes.data
        d.global_count = gmap.global_count
        d.group_offsets = offs.ctypes.data
        d.group_nodes = nodes.ctypes.data
        if mesh is not None and mesh.structured():
            if mesh.elem_count != gf.elem_count:
                raise ContractViolation("HelmholtzOperator: mesh / geometry size mismatch")
            corners = np.ascontiguousarray(mesh.corners, np.float64)
            keep.append(corners)
            d.box[0], d.box[1], d.box[2] = mesh.ex, mesh.ey, mesh.ez
            for q in range(3):
                d.periodic[q] = int(bool(mesh.periodic[q]))
            d.corners = corners.ctypes.data
        h = C.c_void_p()
        _check(lib.sbx_ctx_create(C.byref(d), device, C.byref(h)))
        return cls(h, device)

    @classmethod
    def box(cls, ex, ey, ez, degree, periodic=(False, False, False), deform=0.0,
            origin=(0.0, 0.0, 0.0), lengths=(1.0, 1.0, 1.0), device=0):
        """Product-native setup of a structured (deformed) box."""
        d = L.BoxDesc()
        d.ex, d.ey, d.ez, d.degree = ex, ey, ez, degree
        for q in range(3):
            d.periodic[q] = int(bool(periodic[q]))
            d.origin[q] = origin[q]
            d.lengths[q] = lengths[q]
        d.deform_amplitude = float(deform)
        h = C.c_void_p()
        _check(lib.sbx_ctx_create_box(C.byref(d), device, C.byref(h)))
        return cls(h, device)

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib.sbx_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def new_field(self, device=True):
        if device:
            import torch

            return torch.zeros(self.nodes, dtype=torch.float64, device=f"cuda:{self.device}")
        return np.zeros(self.nodes)

    def _shape_check(self, *fields):
        for f in fields:
            size = f.size if isinstance(f, np.ndarray) else f.numel()
            if size != self.nodes:
                raise ContractViolation("field does not match the operator's grid/shape")

    def array(self, which):
        """copy a context array back (0 mask, 1 inv_mult, 2 bm, 3..8 g1..g6, 9 deriv)."""
        count = self.n1d * self.n1d if which == 9 else self.nodes
        out = np.empty(count)
        _check(lib.sbx_ctx_copy_array(self._h, which, out.ctypes.data))
        return out

    def features(self):
        """{"lattice_gs", "box_k2", "trilinear"}: the fused paths this context runs."""
        f = C.c_uint32()
        _check(lib.sbx_ctx_features(self._h, C.byref(f)))
        names = ((L.FEAT_LATTICE_GS, "lattice_gs"), (L.FEAT_BOX_K2, "box_k2"),
                 (L.FEAT_TRILINEAR, "trilinear"))
        return {nm for bit, nm in names if f.value & bit}

    def enable_timing(self, on=True):
        _check(lib.sbx_ctx_enable_timing(self._h, int(on)))

    def kernel_time(self, name):
        ms, cnt = C.c_double(), C.c_int64()
        _check(lib.sbx_ctx_kernel_time(self._h, name.encode(), C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value


def axhelm(u, coeffs: HelmholtzCoeffs, ctx: Context, out=None, exact=False, flip=False):
    """operators.hpp:57-60 / operators.cpp:215-263 (GeometricFactors and
    SpectralBasis live in ctx)."""
    u = _f64(u)
    ctx._shape_check(u)
    if out is None:
        out = np.empty(ctx.nodes) if isinstance(u, np.ndarray) else u.new_empty(ctx.nodes)
    flags = (L.FLAG_EXACT if exact else 0) | (L.FLAG_FLIP_T if flip else 0)
    with _coeff_fields(ctx, coeffs):
        _check(lib.sbx_axhelm(ctx.handle, _ptr(u), _ptr(out), coeffs.h1, coeffs.h2, flags))
    return out


def debug_cg_k1(u, coeffs: HelmholtzCoeffs, ctx: Context, out=None):
    """Test hook: w = A_local u from the fused solver's own element kernel
    (K1, first-iteration form; the on-the-fly trilinear metric on box
    contexts).  Same result contract as axhelm (operators.cpp:215-263)."""
    u = _f64(u)
    ctx._shape_check(u)
    if out is None:
        out = np.empty(ctx.nodes) if isinstance(u, np.ndarray) else u.new_empty(ctx.nodes)
    _check(lib.sbx_debug_cg_k1(ctx.handle, _ptr(u), _ptr(out), coeffs.h1, coeffs.h2))
    return out


def axhelm_diagonal(coeffs: HelmholtzCoeffs, ctx: Context, assembled=False, device=False):
    """operators.hpp:64-66 / operators.cpp:272-298 (+ gs_sum when assembled)."""
    out = ctx.new_field(device)
    with _coeff_fields(ctx, coeffs):
        _check(lib.sbx_axhelm_diagonal(ctx.handle, coeffs.h1, coeffs.h2, int(assembled),
                                       _ptr(out)))
    return out


def gs_sum_inplace(ctx: Context, f):
    """gather.hpp:39 / gather.cpp:85-98 (bitwise equal)."""
    ctx._shape_check(f)
    _check(lib.sbx_gs_sum(ctx.handle, _ptr(f)))
    return f


def gs_sum(ctx: Context, f):
    """gather.hpp:38"""
    g = f.copy() if isinstance(f, np.ndarray) else f.clone()
    return gs_sum_inplace(ctx, g)


def field_dot_weighted(ctx: Context, a, b, exact=True):
    """field.hpp:60-62 / field.cpp:69-81"""
    ctx._shape_check(a, b)
    out = C.c_double()
    _check(lib.sbx_dot(ctx.handle, _ptr(_f64(a)), _ptr(_f64(b)), 1,
                       L.FLAG_EXACT if exact else 0, C.byref(out)))
    return out.value


def field_dot(ctx: Context, a, b, exact=True):
    """field.hpp:58 / field.cpp:59-67"""
    ctx._shape_check(a, b)
    out = C.c_double()
    _check(lib.sbx_dot(ctx.handle, _ptr(_f64(a)), _ptr(_f64(b)), 0,
                       L.FLAG_EXACT if exact else 0, C.byref(out)))
    return out.value


class HelmholtzOperator:
    """operators.hpp:103-112: A(u) = mask(gs_sum(axhelm(u)))."""

    def __init__(self, ctx: Context, coeffs: HelmholtzCoeffs = HelmholtzCoeffs(),
                 use_mask: bool = True, exact: bool = False):
        self.ctx = ctx
        self.coeffs = coeffs
        self.use_mask = use_mask
        self.exact = exact

    def apply(self, x, out):
        x = _f64(x)
        self.ctx._shape_check(x, out)
        flags = (L.FLAG_EXACT if self.exact else 0) | (0 if self.use_mask else L.FLAG_NO_MASK)
        with _coeff_fields(self.ctx, self.coeffs):
            _check(lib.sbx_apply(self.ctx.handle, _ptr(x), _ptr(out), self.coeffs.h1,
                                 self.coeffs.h2, flags))
        return out

    __call__ = apply

    def assembled_diagonal(self, device=False):
        return axhelm_diagonal(self.coeffs, self.ctx, assembled=True, device=device)


def pcg(op: HelmholtzOperator, b, x, cfg: KrylovConfig = KrylovConfig(),
        precond: Optional[str] = "jacobi", mode: str = "fast", history=True) -> PcgResult:
    """krylov.hpp:38-40 / krylov.cpp:7-91 with ApplyFn = op.apply, DotFn =
    field_dot_weighted and PrecondFn = Jacobi on op.assembled_diagonal() (or
    none).  x is the initial guess in / solution out.  NaN/Inf or breakdown
    raise SolverError(iteration); max_iterations is reported, not raised.
    mode "exact" reproduces the reference bit for bit; "fast" is the fused
    device-resident solver."""
    if not op.use_mask:
        # the fused and the reference-order solvers both solve the masked
        # (Dirichlet) system; the unmasked operator is singular for Poisson
        raise ContractViolation("pcg: HelmholtzOperator(use_mask=False) is not supported")
    b = _f64(b)
    op.ctx._shape_check(b, x)
    c = L.PcgConfig()
    lib.sbx_pcg_config_default(C.byref(c))
    c.tolerance = cfg.tolerance
    c.max_iterations = cfg.max_iterations
    c.precond = L.PRECOND_JACOBI if precond == "jacobi" else L.PRECOND_NONE
    c.mode = L.MODE_EXACT if mode == "exact" else L.MODE_FAST
    c.h1 = op.coeffs.h1
    c.h2 = op.coeffs.h2
    hist = None
    if history:
        hist = np.zeros(max(cfg.max_iterations, 0) + 1)
        c.history = hist.ctypes.data
        c.history_capacity = hist.size
    r = L.PcgResultC()
    with _coeff_fields(op.ctx, op.coeffs):
        rc = lib.sbx_pcg(op.ctx.handle, _ptr(b), _ptr(x), C.byref(c), C.byref(r))
    _check(rc, r.error_iteration)
    out = PcgResult(r.iterations, r.rel_residual, r.rel_residual_precond, bool(r.converged))
    if hist is not None:
        out.residual_history = hist[: min(r.history_length, hist.size)].tolist()
    return out


# ------------------------------------------------ pressure (P_N / P_N-2) ----
@dataclass
class PressureBasis:
    """basis.hpp:21-35"""

    order: int            # N-2
    velocity_order: int   # N
    nodes: np.ndarray     # N-1 GL points
    weights: np.ndarray
    interp_v2p: np.ndarray  # (N-1) x (N+1) row-major

    def m(self):
        return self.order + 1

    def nv(self):
        return self.velocity_order + 1


def build_pressure_basis(velocity_degree: int) -> PressureBasis:
    """basis.hpp:46 / basis.cpp:114-145"""
    m = max(velocity_degree - 1, 1)
    nodes, weights = np.zeros(m), np.zeros(m)
    interp = np.zeros(m * (velocity_degree + 1))
    _check(lib.sbx_pressure_basis(velocity_degree, nodes.ctypes.data, weights.ctypes.data,
                                  interp.ctypes.data))
    return PressureBasis(velocity_degree - 2, velocity_degree, nodes, weights, interp)


def _pnodes(ctx: Context):
    n, m = C.c_int64(), C.c_int32()
    _check(lib.sbx_pressure_info(ctx.handle, C.byref(n), C.byref(m)))
    return n.value


def _pshape(ctx, *fields):
    N = _pnodes(ctx)
    for f in fields:
        size = f.size if isinstance(f, np.ndarray) else f.numel()
        if size != N:
            raise ContractViolation("pressure field does not match the pressure grid")
    return N


def gradient_from_pressure(p, ctx: Context, exact=False):
    """operators.hpp:78-80 / operators.cpp:365-410 -> [gx, gy, gz] (velocity grid);
    exact = the reference's evaluation order (bitwise)."""
    p = _f64(p)
    _pshape(ctx, p)
    if isinstance(p, np.ndarray):
        out = [np.empty(ctx.nodes) for _ in range(3)]
    else:
        out = [p.new_empty(ctx.nodes) for _ in range(3)]
    _check(lib.sbx_gradient_from_pressure(ctx.handle, _ptr(p), *[_ptr(o) for o in out],
                                          L.FLAG_EXACT if exact else 0))
    return out


def divergence_to_pressure(ux, uy, uz, ctx: Context, exact=False):
    """operators.hpp:73-75 / operators.cpp:327-363 (pressure grid)."""
    u = [_f64(v) for v in (ux, uy, uz)]
    ctx._shape_check(*u)
    N = _pnodes(ctx)
    out = np.empty(N) if isinstance(u[0], np.ndarray) else u[0].new_empty(N)
    _check(lib.sbx_divergence_to_pressure(ctx.handle, *[_ptr(v) for v in u], _ptr(out),
                                          L.FLAG_EXACT if exact else 0))
    return out


class PressureOperator:
    """FlowSolver::apply_pressure_operator / pressure_operator_diagonal
    (stepper.cpp:240-275): E p = Div (mask / gs(bm)) gs Grad p."""

    def __init__(self, ctx: Context, exact: bool = False):
        self.ctx = ctx
        self.exact = exact
        self.nodes = _pnodes(ctx)

    def apply(self, p, out):
        p = _f64(p)
        _pshape(self.ctx, p, out)
        _check(lib.sbx_pressure_apply(self.ctx.handle, _ptr(p), _ptr(out),
                                      L.FLAG_EXACT if self.exact else 0))
        return out

    __call__ = apply

    def diagonal(self):
        out = np.empty(self.nodes)
        _check(lib.sbx_pressure_diagonal(self.ctx.handle, out.ctypes.data,
                                         L.FLAG_EXACT if self.exact else 0))
        return out


def pcg_pressure(op: PressureOperator, b, x, cfg: KrylovConfig = KrylovConfig(),
                 precond: Optional[str] = "jacobi", history=True, mode: str = "fast") -> PcgResult:
    """The pressure solve of FlowSolver::solve_pressure_update
    (stepper.cpp:326-347): pcg with the pressure operator, the plain field_dot
    and pressure_precond (Jacobi or none, each with the mean deflation).  b
    must have its mean removed (stepper.cpp:313-324); x is the initial guess
    in / solution out.  mode "exact" reproduces the reference bit for bit,
    "fast" is the fused device loop."""
    b = _f64(b)
    _pshape(op.ctx, b, x)
    c = L.PcgConfig()
    lib.sbx_pcg_config_default(C.byref(c))
    c.tolerance = cfg.tolerance
    c.max_iterations = cfg.max_iterations
    c.precond = L.PRECOND_JACOBI if precond == "jacobi" else L.PRECOND_NONE
    c.mode = L.MODE_EXACT if mode == "exact" else L.MODE_FAST
    hist = None
    if history:
        hist = np.zeros(max(cfg.max_iterations, 0) + 1)
        c.history = hist.ctypes.data
        c.history_capacity = hist.size
    r = L.PcgResultC()
    rc = lib.sbx_pressure_pcg(op.ctx.handle, _ptr(b), _ptr(x), C.byref(c), C.byref(r))
    _check(rc, r.error_iteration)
    out = PcgResult(r.iterations, r.rel_residual, r.rel_residual_precond, bool(r.converged))
    if hist is not None:
        out.residual_history = hist[: min(r.history_length, hist.size)].tolist()
    return out


class ProjectionHistory:
    """krylov.hpp:45-64 / krylov.cpp:93-124 on the pressure grid of ctx (the
    pressure solve's initial-guess projection, stepper.cpp:326 and 345): the
    A-orthonormal (x, E x) pairs stay on the device; plain field_dot."""

    def __init__(self, ctx: Context, depth: int, exact: bool = False):
        self.ctx = ctx
        self.exact = exact
        self.nodes = _pnodes(ctx)
        _check(lib.sbx_projection_reset(ctx.handle, int(depth)))
        self._depth = depth

    def depth(self):
        return self._depth

    def size(self):
        n = C.c_int32()
        _check(lib.sbx_projection_size(self.ctx.handle, C.byref(n)))
        return n.value

    def project_guess(self, b, deflated_rhs=False):
        """guess = sum_i (x_i . b) x_i [, b - E guess]"""
        b = _f64(b)
        _pshape(self.ctx, b)
        new = (lambda: np.empty(self.nodes)) if isinstance(b, np.ndarray) else \
            (lambda: b.new_empty(self.nodes))
        guess = new()
        defl = new() if deflated_rhs else None
        _check(lib.sbx_projection_guess(self.ctx.handle, _ptr(b), _ptr(guess), _ptr(defl),
                                        L.FLAG_EXACT if self.exact else 0))
        return (guess, defl) if deflated_rhs else guess

    def append(self, x):
        x = _f64(x)
        _pshape(self.ctx, x)
        _check(lib.sbx_projection_append(self.ctx.handle, _ptr(x),
                                         L.FLAG_EXACT if self.exact else 0))


def advect(u, c, ctx: Context):
    """operators.hpp:84-87 / operators.cpp:412-431: out_d = bm (c . grad u_d),
    reference evaluation order (bitwise)."""
    u = [_f64(v) for v in u]
    c = [_f64(v) for v in c]
    ctx._shape_check(*u, *c)
    out = [np.empty(ctx.nodes) if isinstance(u[0], np.ndarray) else u[0].new_empty(ctx.nodes)
           for _ in range(3)]
    arr = lambda vs: (C.c_void_p * 3)(*[_ptr(v) for v in vs])  # noqa: E731
    _check(lib.sbx_advect(ctx.handle, arr(u), arr(c), arr(out)))
    return out


def pcg_multi(op: HelmholtzOperator, bs, xs, cfg: KrylovConfig = KrylovConfig(),
              precond: Optional[str] = "jacobi", mode: str = "fast", history=True):
    """FlowSolver::solve_velocity_star's three component solves
    (stepper.cpp:188-238) as one batched call: bs[d], xs[d] (initial guess in,
    solution out), the same operator and KrylovConfig for every component.
    Returns one PcgResult per component."""
    if not op.use_mask:
        raise ContractViolation("pcg: HelmholtzOperator(use_mask=False) is not supported")
    count = len(bs)
    if count != len(xs) or not 1 <= count <= 3:
        raise ContractViolation("pcg_multi: 1 to 3 right-hand sides, one x each")
    bs = [_f64(b) for b in bs]
    op.ctx._shape_check(*bs, *xs)
    c = L.PcgConfig()
    lib.sbx_pcg_config_default(C.byref(c))
    c.tolerance = cfg.tolerance
    c.max_iterations = cfg.max_iterations
    c.precond = L.PRECOND_JACOBI if precond == "jacobi" else L.PRECOND_NONE
    c.mode = L.MODE_EXACT if mode == "exact" else L.MODE_FAST
    c.h1 = op.coeffs.h1
    c.h2 = op.coeffs.h2
    hist = None
    cap = max(cfg.max_iterations, 0) + 1
    if history:
        hist = np.zeros(count * cap)
        c.history = hist.ctypes.data
        c.history_capacity = cap
    res = (L.PcgResultC * count)()
    barr = (C.c_void_p * count)(*[_ptr(b) for b in bs])
    xarr = (C.c_void_p * count)(*[_ptr(x) for x in xs])
    with _coeff_fields(op.ctx, op.coeffs):
        rc = lib.sbx_pcg_multi(op.ctx.handle, count, barr, xarr, C.byref(c), res)
    err_it = max((r.error_iteration for r in res), default=-1)
    _check(rc, err_it)
    out = []
    for d, r in enumerate(res):
        o = PcgResult(r.iterations, r.rel_residual, r.rel_residual_precond, bool(r.converged))
        if hist is not None:
            o.residual_history = hist[d * cap: d * cap + min(r.history_length, cap)].tolist()
        out.append(o)
    return out
