"""B200-native (sm_100a) hot path of the mixed-precision LOBPCG / PINVIT
eigensolver (arXiv 2302.12528), behind the reference library's entry points.

The numerics live in ``libmpeig_b200.so`` (CUDA kernels + C++ driver, C ABI
in ``include/mpeig_b200.h``); this package is the thin Python mirror of the
reference interface used by the tests and the benchmark.
"""
from .api import (  # noqa: F401
    LOWER, WORKING, CallbackError, CommError, ConfigError, Context, CudaError, DimensionMismatch,
    HostGroup, broadcast_unique_id, gaussian_matrix_rows, laplace3d_slab, nccl_unique_id,
    slab_partition,
    EigResult, IterationRecord, MpeigError, NoConvergence, NotPositiveDefinite, Operator,
    OverflowError_, RankCollapse, RankDeficient, SingularTriangular, SolverConfig,
    StageOptions, StageOutcome, StageTimings, build_precision_for, converged_count, csr_matrix, csr_rows,
    default_context, dense_cholesky, dense_matrix, rcm_ordering, solve_csr, sparse_cholesky,
    ks_hamiltonian, ks_hamiltonian_slab, read_matrix_market, ParseError, NotSymmetricHeader, NotSquare, gaussian_matrix, host_operator, jacobi, laplace2d, laplace3d,
    lobpcg_stage, mixed_lobpcg, pinvit, profile, run_variant, solve, solve_prepared,
    spectral_norm_estimate, to_device,
    to_host,
)
from ._lib import LIB_PATH, SYMBOLS, load  # noqa: F401
from . import generators  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
