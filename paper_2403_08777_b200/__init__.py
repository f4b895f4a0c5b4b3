"""B200-native momentum-RHS finite-element assembly on linear tetrahedra.

A drop-in for the hot path of the reference package tet-assembly-lab 0.1.0
(arXiv 2403.08777, Alya nsi element operations): ``assemble_rsp`` and the
numba seam ``assemble_elements`` run as hand-written sm_100a CUDA kernels in
``libtal_b200.so`` behind a C-ABI (include/tal_b200.h).
"""

from .assembly import (
    ASSEMBLERS,
    NULL_SCALE_FRACTION,
    REL_TOL,
    SCATTER_MODES,
    Assembler,
    AssemblyResult,
    CounterLedger,
    RunConfig,
    Timings,
    VARIANT_INFO,
    VariantId,
    VariantCheck,
    VariantInfo,
    VerifyReport,
    assemble,
    assemble_baseline,
    assemble_elements,
    assemble_rs,
    assemble_rsp,
    clear_cache,
    contribution_scale,
    make_ledger,
    oracle_compare,
    verify_variants,
)
from .fields import (
    DENOM_EPSILON,
    INITIALIZERS,
    PhysParams,
    QuadratureRule,
    interpolation_table,
    make_velocity,
    quadrature_tet4,
    validate_velocity,
)
from .mesh import (
    Mesh,
    color_elements,
    generate_box_mesh,
    generate_delaunay_mesh,
    permute_nodes,
    renumber_nodes,
    signed_volumes,
)

__version__ = "0.1.0"
