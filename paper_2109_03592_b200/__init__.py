"""B200-native matrix-free spectral-element PCG (the hot path of
arXiv:2109.03592's Nek5000), behind the reference's ("sembox") operator API.

Compute runs only in the in-tree CUDA library libsbx.so (sm_100a); importing
this package without it raises ImportError.
"""
from .api import (  # noqa: F401
    ConfigError,
    Context,
    ContractViolation,
    CudaError,
    GatherScatterMap,
    GeometricFactors,
    HelmholtzCoeffs,
    HelmholtzOperator,
    HexMesh,
    KrylovConfig,
    MeshError,
    PcgResult,
    PressureBasis,
    PressureOperator,
    ProjectionHistory,
    SemboxError,
    SolverError,
    SpectralBasis,
    advect,
    axhelm,
    axhelm_diagonal,
    debug_cg_k1,
    build_box_mesh,
    build_dirichlet_mask,
    build_gather_scatter,
    build_geometric_factors,
    build_gll_basis,
    build_pressure_basis,
    divergence_to_pressure,
    gradient_from_pressure,
    field_dot,
    field_dot_weighted,
    gs_sum,
    gs_sum_inplace,
    partition_rcb,
    pcg,
    pcg_multi,
    pcg_pressure,
)

__version__ = "0.1.0"
