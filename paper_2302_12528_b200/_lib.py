"""ctypes binding of libmpeig_b200.so (the C ABI in include/mpeig_b200.h).

The product path has no CPU fallback: if the shared library (built by
``__graft_entry__.build()`` / ``make -C paper_2302_12528_b200/csrc``) is
missing or a CUDA device is absent, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmpeig_b200.so")

# ---- status codes (mpeig_status) ------------------------------------------
OK, E_DIMENSION, E_CONFIG, E_NOT_PD, E_SINGULAR_TRI, E_RANK_DEFICIENT = 0, 1, 2, 3, 4, 5
E_RANK_COLLAPSE, E_NO_CONVERGENCE, E_OVERFLOW, E_CALLBACK = 6, 7, 8, 20
E_CUDA, E_CUSOLVER, E_COMM, E_OTHER = 30, 31, 32, 99

WORKING, LOWER = 0, 1
VARIANTS = {"dlobpcg-dchol": 0, "dlobpcg-schol": 1, "mplobpcg-schol": 2, "pinvit": 3}


class Cfg(C.Structure):
    _fields_ = [("k", C.c_int64), ("block", C.c_int64), ("maxit", C.c_int64),
                ("tol", C.c_double), ("lower_tol", C.c_double), ("seed", C.c_uint64),
                ("variant", C.c_int32), ("sketch_rows", C.c_int64)]


class StageOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("use_mixed_qr", C.c_int32),
                ("stagnation_exit", C.c_int32), ("tag", C.c_int32)]


class IterRecord(C.Structure):
    _fields_ = [("stage", C.c_int32), ("m", C.c_int64),
                ("ritz_values", C.POINTER(C.c_double)),
                ("residual_norms", C.POINTER(C.c_double)),
                ("n_converged", C.c_int64), ("w_columns_dropped", C.c_int64),
                ("basis_rotation_fallback", C.c_int32)]


class Timings(C.Structure):
    _fields_ = [("factorize", C.c_double), ("precond_apply", C.c_double),
                ("orthogonalize", C.c_double), ("projected_eig", C.c_double),
                ("total", C.c_double)]


class StageOut(C.Structure):
    _fields_ = [("X", C.c_void_p), ("ldx", C.c_int64), ("theta", C.POINTER(C.c_double)),
                ("residual_norms", C.POINTER(C.c_double)), ("iterations", C.c_int64),
                ("converged", C.c_int32)]


class Result(C.Structure):
    _fields_ = [("theta", C.POINTER(C.c_double)), ("residual_norms", C.POINTER(C.c_double)),
                ("X", C.c_void_p), ("ldx", C.c_int64), ("iterations_lower", C.c_int64),
                ("iterations_working", C.c_int64), ("converged", C.c_int32),
                ("a_norm_estimate", C.c_double), ("timings", Timings)]


SINK = C.CFUNCTYPE(None, C.c_void_p, C.POINTER(IterRecord))
DEV_APPLY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_int64,
                        C.c_void_p, C.c_int64, C.c_void_p)
HOST_APPLY = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p)

# exported symbols declared by include/mpeig_b200.h (checked by tests)
SYMBOLS = [
    "mpeig_ctx_create", "mpeig_ctx_destroy", "mpeig_last_error", "mpeig_launch_count",
    "mpeig_ctx_stream", "mpeig_ctx_set_option", "mpeig_spec_rollbacks", "mpeig_op_lap3d", "mpeig_op_lap3d_diag", "mpeig_op_lap3d_slab_diag", "mpeig_op_lap2d", "mpeig_op_csr", "mpeig_op_csr_rows", "mpeig_op_dense",
    "mpeig_op_device_callback", "mpeig_op_host_callback", "mpeig_precond_jacobi", "mpeig_precond_dense_chol", "mpeig_precond_shift",
    "mpeig_precond_sparse_chol", "mpeig_precond_factor_nnz", "mpeig_rcm_ordering",
    "mpeig_op_destroy", "mpeig_op_n", "mpeig_op_apply", "mpeig_spectral_norm_estimate",
    "mpeig_lobpcg_stage_f64", "mpeig_lobpcg_stage_f32", "mpeig_pinvit_f64", "mpeig_solve",
    "mpeig_run_variant", "mpeig_gaussian_matrix_host", "mpeig_orthonormal_q_f64",
    "mpeig_orthonormal_q_f32", "mpeig_mixed_qr_f64", "mpeig_householder_qr_f64",
    "mpeig_orthonormal_q_dropping_f64", "mpeig_gram_f64", "mpeig_gemm_f64",
    "mpeig_project_out_f64", "mpeig_small_eig_f64", "mpeig_hl_coeffs_f64",
    "mpeig_residual_precond_f64", "mpeig_solve_prepared", "mpeig_solve_csr",
    "mpeig_buffer_alloc", "mpeig_buffer_free", "mpeig_copy", "mpeig_gram_f32", "mpeig_gemm_f32",
    "mpeig_set_process_option", "mpeig_profile_enable",
    "mpeig_profile_reset", "mpeig_profile_names", "mpeig_profile_query",
    "mpeig_nccl_unique_id", "mpeig_ctx_attach_nccl", "mpeig_host_group_create",
    "mpeig_host_group_destroy", "mpeig_ctx_attach_host_comm", "mpeig_op_lap3d_slab",
    "mpeig_gaussian_matrix_rows_host",
]

_lib = None


def load() -> C.CDLL:
    """Load libmpeig_b200.so and declare signatures (raises if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with __graft_entry__.build() "
                          "(no CPU fallback exists for this path)")
    lib = C.CDLL(LIB_PATH)
    vp, i64, i32, dbl, u64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64
    pvp = C.POINTER(C.c_void_p)
    sig = {
        "mpeig_ctx_create": (C.c_int, [C.c_int, vp, pvp]),
        "mpeig_ctx_destroy": (None, [vp]),
        "mpeig_last_error": (C.c_char_p, [vp, C.POINTER(i64)]),
        "mpeig_launch_count": (i64, [vp, C.c_int]),
        "mpeig_spec_rollbacks": (i64, [vp, C.c_int]),
        "mpeig_ctx_stream": (vp, [vp]),
        "mpeig_ctx_set_option": (C.c_int, [vp, C.c_char_p, C.c_int]),
        "mpeig_op_lap3d": (C.c_int, [vp, i64, i64, i64, pvp]),
        "mpeig_op_lap2d": (C.c_int, [vp, i64, i64, pvp]),
        "mpeig_op_csr": (C.c_int, [vp, i64, vp, vp, vp, pvp]),
        "mpeig_op_csr_rows": (C.c_int, [vp, i64, i64, i64, vp, vp, vp, pvp]),
        "mpeig_op_dense": (C.c_int, [vp, i64, vp, i64, pvp]),
        "mpeig_op_device_callback": (C.c_int, [vp, i64, DEV_APPLY, DEV_APPLY, vp, pvp]),
        "mpeig_op_host_callback": (C.c_int, [vp, i64, HOST_APPLY, HOST_APPLY, vp, pvp]),
        "mpeig_precond_jacobi": (C.c_int, [vp, vp, i32, pvp]),
        "mpeig_precond_dense_chol": (C.c_int, [vp, vp, i32, pvp]),
        "mpeig_precond_shift": (C.c_double, [vp]),
        "mpeig_precond_sparse_chol": (C.c_int, [vp, vp, i32, i32, vp, pvp]),
        "mpeig_precond_factor_nnz": (i64, [vp]),
        "mpeig_rcm_ordering": (C.c_int, [i64, vp, vp, vp]),
        "mpeig_op_destroy": (None, [vp]),
        "mpeig_op_n": (i64, [vp]),
        "mpeig_op_apply": (C.c_int, [vp, vp, i32, i64, vp, i64, vp, i64]),
        "mpeig_spectral_norm_estimate": (C.c_int, [vp, vp, i64, u64, C.POINTER(dbl)]),
        "mpeig_lobpcg_stage_f64": (C.c_int, [vp, vp, i64, vp, i64, i64, C.POINTER(Cfg), vp, dbl,
                                             C.POINTER(StageOpts), SINK, vp, C.POINTER(StageOut),
                                             C.POINTER(Timings)]),
        "mpeig_lobpcg_stage_f32": (C.c_int, [vp, vp, i64, vp, i64, i64, C.POINTER(Cfg), vp, dbl,
                                             C.POINTER(StageOpts), SINK, vp, C.POINTER(StageOut),
                                             C.POINTER(Timings)]),
        "mpeig_pinvit_f64": (C.c_int, [vp, vp, i64, vp, i64, i64, C.POINTER(Cfg), vp, dbl, SINK,
                                       vp, C.POINTER(Result)]),
        "mpeig_solve": (C.c_int, [vp, vp, vp, C.POINTER(Cfg), SINK, vp, C.POINTER(Result)]),
        "mpeig_run_variant": (C.c_int, [vp, vp, vp, C.POINTER(Cfg), vp, i64, dbl, SINK, vp,
                                        C.POINTER(Result)]),
        "mpeig_gaussian_matrix_host": (C.c_int, [i64, i64, u64, vp]),
        "mpeig_gaussian_matrix_rows_host": (C.c_int, [i64, i64, u64, i64, i64, vp]),
        "mpeig_orthonormal_q_f64": (C.c_int, [vp, i64, i64, vp, i64, i32]),
        "mpeig_orthonormal_q_f32": (C.c_int, [vp, i64, i64, vp, i64]),
        "mpeig_mixed_qr_f64": (C.c_int, [vp, i64, i64, vp, i64, vp]),
        "mpeig_householder_qr_f64": (C.c_int, [vp, i64, i64, vp, i64, vp]),
        "mpeig_orthonormal_q_dropping_f64": (C.c_int, [vp, i64, i64, vp, i64, i32, C.POINTER(i64)]),
        "mpeig_gram_f64": (C.c_int, [vp, i64, i64, vp, i64, i64, vp, i64, vp]),
        "mpeig_gemm_f64": (C.c_int, [vp, i64, i64, i64, dbl, vp, i64, vp, i64, dbl, vp, i64, vp,
                                     i64]),
        "mpeig_set_process_option": (C.c_int, [C.c_char_p, C.c_int]),
        "mpeig_op_lap3d_diag": (C.c_int, [vp, i64, i64, i64, vp, pvp]),
        "mpeig_op_lap3d_slab_diag": (C.c_int, [vp, i64, i64, i64, i64, i64, vp, pvp]),
        "mpeig_gram_f32": (C.c_int, [vp, i64, i64, vp, i64, i64, vp, i64, vp]),
        "mpeig_gemm_f32": (C.c_int, [vp, i64, i64, i64, C.c_float, vp, i64, vp, i64, C.c_float, vp,
                                     i64, vp, i64]),
        "mpeig_project_out_f64": (C.c_int, [vp, i64, i64, vp, i64, i64, vp, i64, i32]),
        "mpeig_small_eig_f64": (C.c_int, [vp, i64, vp, vp, vp]),
        "mpeig_hl_coeffs_f64": (C.c_int, [vp, i64, i64, vp, vp, C.POINTER(i64), C.POINTER(i32)]),
        "mpeig_residual_precond_f64": (C.c_int, [vp, vp, i64, i64, vp, i64, vp, i64, vp, vp, i64,
                                                 vp, vp]),
        "mpeig_solve_prepared": (C.c_int, [vp, vp, vp, C.POINTER(Cfg), vp, i64, vp, i64, dbl, SINK,
                                           vp, C.POINTER(Result)]),
        "mpeig_solve_csr": (C.c_int, [vp, i64, vp, vp, vp, C.POINTER(Cfg), SINK, vp,
                                      C.POINTER(Result), C.POINTER(dbl)]),
        "mpeig_buffer_alloc": (C.c_int, [vp, i64, pvp]),
        "mpeig_buffer_free": (None, [vp, vp]),
        "mpeig_copy": (C.c_int, [vp, vp, vp, i64]),
        "mpeig_nccl_unique_id": (C.c_int, [vp, i64]),
        "mpeig_ctx_attach_nccl": (C.c_int, [vp, C.c_int, C.c_int, vp]),
        "mpeig_host_group_create": (C.c_int, [C.c_int, pvp]),
        "mpeig_host_group_destroy": (None, [vp]),
        "mpeig_ctx_attach_host_comm": (C.c_int, [vp, vp, C.c_int]),
        "mpeig_op_lap3d_slab": (C.c_int, [vp, i64, i64, i64, i64, i64, pvp]),
        "mpeig_profile_enable": (None, [C.c_int]),
        "mpeig_profile_reset": (None, []),
        "mpeig_profile_names": (C.c_int, [C.c_char_p, i64]),
        "mpeig_profile_query": (C.c_int, [C.c_char_p, C.POINTER(i64), C.POINTER(dbl),
                                          C.POINTER(dbl), C.POINTER(dbl)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
