"""hexbp-b200: B200-native matrix-free BP operator + CG hot path.

A drop-in for the reference hexbp operator apply / CG path
(/root/reference/proj/include/hexbp/operator.hpp, solver.hpp): one fused
sm_100a kernel per operator apply (restriction gather, sum-factorised
B/D contractions, streamed geometric factors, deterministic transpose
restriction), device-resident CG with fused vector updates, C ABI in
include/hexbp_b200.h.
"""
from .api import (  # noqa: F401
    Backend,
    BCSet,
    BPKind,
    CGReport,
    ConstrainedOperator,
    DegenerateElementError,
    DivergenceError,
    FlopCount,
    HexbpCudaError,
    HexMesh,
    OperatorHandle,
    OperatorSetup,
    Workspace,
    bench_rhs,
    boundary_bcs,
    boundary_nodes,
    build_box_mesh,
    cg,
    default_quad_points,
    degenerate_element_error,
    device_count,
    divergence_error,
    is_diffusion,
    jacobi_diagonal,
    make_operator,
    make_setup,
    make_slab_setup,
    parse_backend,
    parse_bp,
    to_string,
)

__all__ = [n for n in dir() if not n.startswith("_")]
from .fe import (  # noqa: F401,E402
    assemble_load,
    boundary_mask,
    discrete_l2_error,
    factors_device,
    interp_to_qpts,
    interp_transpose,
    nodal_interpolant,
    node_coords,
    quadrature_points,
)
