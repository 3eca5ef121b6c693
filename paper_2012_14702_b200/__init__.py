"""B200-native iterative perturbation theory (IPT, arXiv 2012.14702) hot path.

The drop-in boundary is the C ABI in include/ipt_cuda.h (libipt_b200.so); this
package is the Python mirror of the reference's C++ solver API on top of it.
"""
from .ipt import (  # noqa: F401
    Context,
    CsrMatrix,
    DegenerateDiagonal,
    EigenpairResult,
    InverseGaps,
    IterationConfig,
    LuFactors,
    Partition,
    SolveStatus,
    SpectrumResult,
    apply_map_full,
    apply_map_single,
    build_gaps,
    default_context,
    kernels,
    lu_factor,
    lu_solve,
    lu_solve_adjoint,
    lu_solve_matrix,
    nccl_unique_id,
    partition,
    reconstruct,
    smallest_singular_value_estimate,
    solve_full,
    solve_single,
    solve_single_accelerated,
    solve_single_continuation,
    to_string,
)
from ._lib import LIB_PATH, IptError, load as load_library  # noqa: F401
