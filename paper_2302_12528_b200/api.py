"""Python mirror of the reference solver interface, backed by the sm_100a C ABI.

Names, argument meaning and error behaviour follow the reference library
(``/root/reference/proj/include/mpeig``):

=============================  ===============================================
this module                    reference
=============================  ===============================================
``SolverConfig``               ``SolverConfig``      solver_types.hpp:31-57
``StageOptions``               ``StageOptions``      eigensolvers.hpp:176-181
``IterationRecord``            ``IterationRecord``   solver_types.hpp:59-66
``StageTimings``               ``StageTimings``      solver_types.hpp:68-74
``EigResult``                  ``EigResult<T>``      solver_types.hpp:76-88
``lobpcg_stage``               ``lobpcg_stage<T>``   eigensolvers.hpp:195-321
``pinvit``                     ``pinvit<T>``         eigensolvers.hpp:326-390
``mixed_lobpcg``               ``mixed_lobpcg``      drivers.hpp:122-152
``solve``                      ``solve``             drivers.hpp:158-210
``jacobi``                     diagonal f_T (the north star's preconditioner)
``dense_cholesky``             ``Preconditioner<T>::build(DenseMatrix, prec)``
                               precond.hpp:33-50 (pass as ``T=`` for the
                               reference's stock dense ``solve``)
``spectral_norm_estimate``     norm_estimate.hpp:15-24
``converged_count``            eigensolvers.hpp:25-43
exceptions                     errors.hpp:10-62
=============================  ===============================================

Device block vectors are torch CUDA tensors used as plain device memory: an
n x m column-major block is a contiguous tensor of shape (m, ld) (row j =
column j).  All numerical work happens in libmpeig_b200.so; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib as L

# ----------------------------------------------------------------- errors


class MpeigError(Exception):
    code = L.E_OTHER

    def __init__(self, msg="", index=-1):
        super().__init__(msg)
        self.index = index


class DimensionMismatch(MpeigError, ValueError):
    code = L.E_DIMENSION


class ConfigError(MpeigError, ValueError):
    code = L.E_CONFIG


class NotPositiveDefinite(MpeigError, RuntimeError):
    code = L.E_NOT_PD


class SingularTriangular(MpeigError, RuntimeError):
    code = L.E_SINGULAR_TRI


class RankDeficient(MpeigError, RuntimeError):
    code = L.E_RANK_DEFICIENT

    @property
    def column(self):
        return self.index


class RankCollapse(MpeigError, RuntimeError):
    code = L.E_RANK_COLLAPSE


class NoConvergence(MpeigError, RuntimeError):
    code = L.E_NO_CONVERGENCE


class OverflowError_(MpeigError, ArithmeticError):
    """OverflowError (errors.hpp:55): a finite value left the binary32 range."""
    code = L.E_OVERFLOW


class CallbackError(MpeigError, RuntimeError):
    code = L.E_CALLBACK


class CudaError(MpeigError, RuntimeError):
    code = L.E_CUDA


class CommError(MpeigError, RuntimeError):
    code = 32  # MPEIG_E_COMM


_ERRORS = {c.code: c for c in (DimensionMismatch, ConfigError, NotPositiveDefinite,
                               SingularTriangular, RankDeficient, RankCollapse, NoConvergence,
                               OverflowError_, CallbackError, CudaError, CommError)}

# ----------------------------------------------------------------- types

WORKING, LOWER = L.WORKING, L.LOWER


@dataclass
class SolverConfig:
    k: int = 1
    block: int = 0
    maxit: int = 2000
    tol: float = 1e-12
    lower_tol: float = 5e-6
    seed: int = 0
    variant: str = "mplobpcg-schol"
    sketch_rows: int = 8

    def block_size(self) -> int:
        return self.block if self.block != 0 else (3 * self.k + 1) // 2

    def to_c(self) -> L.Cfg:
        return L.Cfg(self.k, self.block, self.maxit, self.tol, self.lower_tol,
                     self.seed & 0xFFFFFFFFFFFFFFFF, L.VARIANTS[self.variant], self.sketch_rows)


@dataclass
class StageOptions:
    tol: float = 1e-12
    use_mixed_qr: bool = False
    stagnation_exit: bool = False
    tag: int = WORKING


@dataclass
class IterationRecord:
    stage: int
    ritz_values: List[float]
    residual_norms: List[float]
    n_converged: int
    w_columns_dropped: int
    basis_rotation_fallback: bool
    host_time: float = 0.0  # time.perf_counter() when the record reached the host (diagnostic)


@dataclass
class StageTimings:
    factorize: float = 0.0
    precond_apply: float = 0.0
    orthogonalize: float = 0.0
    projected_eig: float = 0.0
    total: float = 0.0


@dataclass
class EigResult:
    theta: np.ndarray
    X: Optional[object]
    residual_norms: np.ndarray
    iterations_lower: int
    iterations_working: int
    history: List[IterationRecord] = field(default_factory=list)
    converged: bool = False
    timings: StageTimings = field(default_factory=StageTimings)
    a_norm_estimate: float = 0.0


@dataclass
class StageOutcome:
    X: object
    theta: np.ndarray
    residual_norms: np.ndarray
    iterations: int
    converged: bool


# ----------------------------------------------------------------- context


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2302_12528_b200 needs a CUDA device (no CPU fallback)")
    return torch


class Context:
    """One library context per (GPU, stream); ordered on torch's current stream."""

    def __init__(self, device: int = 0, stream=None):
        torch = _torch()
        self.lib = L.load()
        self.device = device
        with torch.cuda.device(device):
            s = stream if stream is not None else torch.cuda.current_stream(device)
        self.torch_stream = s
        h = C.c_void_p()
        rc = self.lib.mpeig_ctx_create(device, C.c_void_p(s.cuda_stream), C.byref(h))
        if rc != 0:
            raise CudaError(f"mpeig_ctx_create failed ({rc})")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.mpeig_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def check(self, rc: int):
        if rc == 0:
            return
        idx = C.c_int64(-1)
        msg = self.lib.mpeig_last_error(self.h, C.byref(idx))
        msg = msg.decode(errors="replace") if msg else ""
        raise _ERRORS.get(rc, MpeigError)(msg, idx.value)

    def set_option(self, key: str, value: int):
        """spec_mode / use_graphs / eig_backend (see include/mpeig_b200.h)."""
        self.check(self.lib.mpeig_ctx_set_option(self.h, key.encode(), int(value)))

    def launches(self, reset=False) -> int:
        return int(self.lib.mpeig_launch_count(self.h, 1 if reset else 0))

    def spec_rollbacks(self, reset=False) -> int:
        """Speculative iterations repeated on the careful path since creation / reset."""
        return int(self.lib.mpeig_spec_rollbacks(self.h, 1 if reset else 0))

    # -- row sharding: rank r solves its rows; see include/mpeig_b200.h
    def attach_nccl(self, rank: int, nranks: int, unique_id: bytes):
        """NCCL communicator over the ranks' GPUs (one process per GPU)."""
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self.check(self.lib.mpeig_ctx_attach_nccl(self.h, int(rank), int(nranks), buf))

    def attach_host(self, group: "HostGroup", rank: int):
        """Rank `rank` of a HostGroup (ranks as threads of this process)."""
        self._group = group  # keep alive
        self.check(self.lib.mpeig_ctx_attach_host_comm(self.h, group.h, int(rank)))


class HostGroup:
    """A group of ranks running as threads of one process; exchanges are
    staged through host memory and reduced in rank order (deterministic)."""

    def __init__(self, nranks: int):
        self.lib = L.load()
        h = C.c_void_p()
        if self.lib.mpeig_host_group_create(int(nranks), C.byref(h)) != 0:
            raise ConfigError("host group: bad size")
        self.h, self.nranks = h, nranks

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.mpeig_host_group_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId (rank 0); broadcast it to the other ranks."""
    lib = L.load()
    buf = C.create_string_buffer(128)
    rc = lib.mpeig_nccl_unique_id(buf, 128)
    if rc != 0:
        raise CommError("NCCL unavailable", -1)
    return buf.raw


def gaussian_matrix_rows(n_global: int, cols: int, seed: int, row0: int, rows: int) -> np.ndarray:
    """Rows [row0, row0 + rows) of gaussian_matrix(n_global, cols, seed)."""
    lib = L.load()
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    rc = lib.mpeig_gaussian_matrix_rows_host(n_global, cols, seed, row0, rows,
                                             out.ctypes.data_as(C.c_void_p))
    if rc != 0:
        raise ConfigError("gaussian_matrix_rows: bad row range", -1)
    return out


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """NCCL id from rank 0 to every rank through torch.distributed (any
    backend, e.g. gloo), for Context.attach_nccl."""
    import torch
    import torch.distributed as dist_
    on_gpu = dist_.get_backend(group) == "nccl"
    buf = torch.zeros(128, dtype=torch.uint8,
                      device=f"cuda:{torch.cuda.current_device()}" if on_gpu else "cpu")
    if rank == 0:
        buf[:] = torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8).to(buf.device)
    dist_.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().tolist())


def slab_partition(nz: int, nranks: int):
    """Balanced z-slabs [(z0, nz_local)] in rank order (rank r holds slab r)."""
    base, extra = divmod(nz, nranks)
    out, z0 = [], 0
    for r in range(nranks):
        nl = base + (1 if r < extra else 0)
        out.append((z0, nl))
        z0 += nl
    return out


_default_ctx: dict = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


# ----------------------------------------------------------------- operators


class Operator:
    """Handle to a device block operator (BlockOperator<T>, dense_kernels.hpp:15-16)."""

    def __init__(self, ctx: Context, handle: C.c_void_p, n: int, kind: str, keep=()):
        self.ctx, self.h, self.n, self.kind = ctx, handle, n, kind
        self._keep = keep  # keeps ctypes callbacks alive

    def __del__(self):
        try:
            if self.h:
                self.ctx.lib.mpeig_op_destroy(self.h)
        except Exception:
            pass

    def apply(self, X, Y=None, precision=WORKING):
        """Y = A X for a device block X (torch tensor of shape (ncols, ld))."""
        torch = _torch()
        ncols, ldx = X.shape
        if Y is None:
            Y = torch.empty_like(X)
        self.ctx.check(self.ctx.lib.mpeig_op_apply(self.ctx.h, self.h, precision, ncols,
                                                   C.c_void_p(X.data_ptr()), ldx,
                                                   C.c_void_p(Y.data_ptr()), Y.shape[1]))
        return Y


def _mk(ctx, fn, *args):
    h = C.c_void_p()
    ctx.check(fn(ctx.h, *args, C.byref(h)))
    return h


def laplace3d(nx: int, ny: int = None, nz: int = None, ctx: Context = None) -> Operator:
    """3-D 7-point Dirichlet Laplacian (diag 6, off -1), row = x + nx (y + ny z)."""
    ctx = ctx or default_context()
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    return Operator(ctx, _mk(ctx, ctx.lib.mpeig_op_lap3d, nx, ny, nz), nx * ny * nz, "lap3d")


def ks_hamiltonian(nx: int, ny: int = None, nz: int = None, seed: int = 0, ctx: Context = None,
                   **kw) -> Operator:
    """cfg5's Kohn-Sham-like H = -Laplacian_7pt + V (generators.ks_potential)
    as a matrix-free stencil with a variable diagonal (mpeig_op_lap3d_diag)."""
    from .generators import ks_diagonal
    ctx = ctx or default_context()
    ny = nx if ny is None else ny
    nz = nx if nz is None else nz
    d = np.ascontiguousarray(ks_diagonal(nx, ny, nz, seed=seed, **kw), dtype=np.float64)
    h = _mk(ctx, ctx.lib.mpeig_op_lap3d_diag, nx, ny, nz, d.ctypes.data)
    return Operator(ctx, h, nx * ny * nz, "ks")


def ks_hamiltonian_slab(nx: int, ny: int, nz_global: int, z0: int, nz_local: int, seed: int = 0,
                        ctx: Context = None, **kw) -> Operator:
    """This rank's z-slab of cfg5's H = -Laplacian_7pt + V (row-sharded)."""
    from .generators import ks_diagonal
    ctx = ctx or default_context()
    d = ks_diagonal(nx, ny, nz_global, seed=seed, **kw)
    row0, n = nx * ny * z0, nx * ny * nz_local
    dl = np.ascontiguousarray(d[row0:row0 + n], dtype=np.float64)
    h = _mk(ctx, ctx.lib.mpeig_op_lap3d_slab_diag, nx, ny, nz_global, z0, nz_local, dl.ctypes.data)
    return Operator(ctx, h, n, "ks_slab")


def laplace3d_slab(nx: int, ny: int, nz_global: int, z0: int, nz_local: int,
                   ctx: Context = None) -> Operator:
    """This rank's z-slab of the 7-point Laplacian (row-sharded; the context
    must be attached to a communicator for more than one rank)."""
    ctx = ctx or default_context()
    h = _mk(ctx, ctx.lib.mpeig_op_lap3d_slab, nx, ny, nz_global, z0, nz_local)
    return Operator(ctx, h, nx * ny * nz_local, "lap3d_slab")


def laplace2d(nx: int, ny: int = None, ctx: Context = None) -> Operator:
    """gen_laplace2d (generators.cpp:13-30) applied matrix-free."""
    ctx = ctx or default_context()
    ny = nx if ny is None else ny
    return Operator(ctx, _mk(ctx, ctx.lib.mpeig_op_lap2d, nx, ny), nx * ny, "lap2d")


def csr_matrix(row_ptr, col_idx, vals, ctx: Context = None) -> Operator:
    """CsrMatrix<double> (csr_matrix.hpp:13-146); columns sorted per row."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    v = np.ascontiguousarray(vals, np.float64)
    n = len(rp) - 1
    h = _mk(ctx, ctx.lib.mpeig_op_csr, n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data)
    return Operator(ctx, h, n, "csr")


def csr_rows(n_global: int, row0: int, row_ptr, col_idx, vals, ctx: Context = None) -> Operator:
    """This rank's row block [row0, row0 + n_local) of a row-sharded CSR matrix
    (global column indices; collective over the context's communicator --
    ghost rows exchanged per apply)."""
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(row_ptr, np.int64)
    ci = np.ascontiguousarray(col_idx, np.int64)
    v = np.ascontiguousarray(vals, np.float64)
    n = len(rp) - 1
    h = _mk(ctx, ctx.lib.mpeig_op_csr_rows, n_global, row0, n, rp.ctypes.data, ci.ctypes.data,
            v.ctypes.data)
    return Operator(ctx, h, n, "csr_rows")


def dense_matrix(A, ctx: Context = None) -> Operator:
    """Dense symmetric operator (herm_product, dense_kernels.hpp:66-72)."""
    ctx = ctx or default_context()
    A = np.asfortranarray(A, dtype=np.float64)
    n = A.shape[0]
    h = _mk(ctx, ctx.lib.mpeig_op_dense, n, A.ctypes.data, n)
    return Operator(ctx, h, n, "dense")


def host_operator(n: int, apply_working: Callable, apply_lower: Callable = None,
                  ctx: Context = None) -> Operator:
    """Wrap a CPU BlockOperator (numpy n x c column-major in -> out)."""
    ctx = ctx or default_context()

    def wrap(fn, dtype):
        if fn is None:
            return L.HOST_APPLY()

        def cb(user, nn, nc, xp, yp):
            try:
                X = np.ctypeslib.as_array(C.cast(xp, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                          shape=(nc * nn,)).reshape((nn, nc), order="F")
                Y = np.asarray(fn(X), dtype=dtype)
                out = np.ctypeslib.as_array(C.cast(yp, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                            shape=(nc * nn,)).reshape((nn, nc), order="F")
                out[...] = Y
                return 0
            except Exception:  # surfaced as CallbackError
                return 1
        return L.HOST_APPLY(cb)

    fw, fl = wrap(apply_working, np.float64), wrap(apply_lower, np.float32)
    h = _mk(ctx, ctx.lib.mpeig_op_host_callback, n, fw, fl, None)
    return Operator(ctx, h, n, "host", keep=(fw, fl))


def jacobi(A: Operator, precision: int = LOWER) -> Operator:
    """Jacobi f_T = diag(A)^-1 built at `precision` (Preconditioner::build)."""
    h = _mk(A.ctx, A.ctx.lib.mpeig_precond_jacobi, A.h, precision)
    return Operator(A.ctx, h, A.n, "jacobi")


def dense_cholesky(A: Operator, precision: int = LOWER) -> Operator:
    """Dense Cholesky f_T = L^-T L^-1 (Preconditioner<T>::build(DenseMatrix, prec),
    precond.hpp:33-50): fp64 factor at WORKING, fp32 factor of to_lower(A) at
    LOWER with retry_dense's one shifted retry (:140-146).  `A` must be a
    dense_matrix() operator.  `.shift` mirrors Preconditioner::shift_applied()."""
    h = _mk(A.ctx, A.ctx.lib.mpeig_precond_dense_chol, A.h, precision)
    op = Operator(A.ctx, h, A.n, "dense_chol", keep=(A,))
    op.shift = float(A.ctx.lib.mpeig_precond_shift(h))
    return op


class ParseError(MpeigError, ValueError):
    """matrix_market.cpp ParseError(line, col, msg)."""

    def __init__(self, line, col, msg):
        super().__init__(f"{line}:{col}: {msg}")
        self.line, self.col = line, col


class NotSymmetricHeader(MpeigError, ValueError):
    """matrix_market.cpp NotSymmetricHeader: only symmetric real input is accepted."""


class NotSquare(MpeigError, ValueError):
    """matrix_market.cpp NotSquare."""


def read_matrix_market(path: str):
    """read_matrix_market_real (matrix_market.cpp:128-157, 204-215) -> (row_ptr, col_idx,
    vals) CSR: banner `%%MatrixMarket matrix coordinate real symmetric` (case-insensitive),
    %-comments and blank lines skipped, 1-based entries mirrored across the diagonal,
    duplicates accumulated (CsrMatrix::from_triplets, csr_matrix.hpp:31-58), columns
    ascending.  Host-side ingestion; feed the result to csr_matrix() or solve_csr()."""
    try:
        f = open(path)
    except OSError:
        raise ParseError(0, 0, f"cannot open '{path}'")
    with f:
        lines = f.read().split("\n")
    if not lines or not lines[0].strip():
        raise ParseError(1, 1, "empty file")
    tok = lines[0].split()
    low = [t.lower() for t in tok]
    if not low or low[0] != "%%matrixmarket":
        raise ParseError(1, 1, "missing %%MatrixMarket banner")
    if len(low) < 2 or low[1] != "matrix":
        raise ParseError(1, 1, "object must be 'matrix'")
    if len(low) < 3 or low[2] != "coordinate":
        raise ParseError(1, 1, "format must be 'coordinate'")
    field = low[3] if len(low) > 3 else ""
    sym = low[4] if len(low) > 4 else ""
    if field != "real":
        raise ParseError(1, 1, f"'{path}' is not a real matrix")
    if sym != "symmetric":
        raise NotSymmetricHeader(sym)
    ln = 1
    size = None
    while ln < len(lines):
        t = lines[ln]
        ln += 1
        if t.startswith("%") or not t.strip():
            continue
        parts = t.split()
        if len(parts) != 3:
            raise ParseError(ln, 1, "expected rows cols nnz")
        try:
            rows, cols, nnz = (int(x) for x in parts)
        except ValueError:
            raise ParseError(ln, 1, "expected an integer")
        if rows != cols:
            raise NotSquare(f"matrix is {rows}x{cols}")
        if rows < 0 or nnz < 0:
            raise ParseError(ln, 1, "negative size")
        size = (rows, nnz)
        break
    if size is None:
        raise ParseError(ln + 1, 1, "missing size line")
    n, nnz = size
    I, J, V = [], [], []
    seen = 0
    while ln < len(lines):
        t = lines[ln]
        ln += 1
        if t.startswith("%") or not t.strip():
            continue
        parts = t.split()
        if len(parts) != 3:
            raise ParseError(ln, 1, "expected i j value")
        try:
            i, j = int(parts[0]), int(parts[1])
        except ValueError:
            raise ParseError(ln, 1, "expected an integer")
        try:
            v = float(parts[2])
        except ValueError:
            raise ParseError(ln, 1, "expected a number")
        if i < 1 or i > n or j < 1 or j > n:
            raise ParseError(ln, 1, "index out of range")
        seen += 1
        if seen > nnz:
            raise ParseError(ln, 1, "more entries than declared")
        I.append(i - 1), J.append(j - 1), V.append(v)
        if i != j:
            I.append(j - 1), J.append(i - 1), V.append(v)
    if seen != nnz:
        raise ParseError(ln + 1, 1, "fewer entries than declared")
    I, J, V = np.array(I, np.int64), np.array(J, np.int64), np.array(V, np.float64)
    order = np.lexsort((J, I))  # stable: duplicates summed in file order
    I, J, V = I[order], J[order], V[order]
    if I.size:
        new = np.ones(I.size, bool)
        new[1:] = (I[1:] != I[:-1]) | (J[1:] != J[:-1])
        idx = np.cumsum(new) - 1
        vals = np.zeros(int(idx[-1]) + 1)
        for q in range(I.size):  # sequential accumulation (from_triplets order)
            vals[idx[q]] += V[q]
        I, J = I[new], J[new]
    else:
        vals = V
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, I + 1, 1)
    return np.cumsum(rp), J, vals


def rcm_ordering(row_ptr, col_idx) -> np.ndarray:
    """rcm_ordering_pattern (rcm.cpp:8-57): perm[k] = original index of row k."""
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    n = rp.size - 1
    perm = np.empty(n, np.int64)
    rc = L.load().mpeig_rcm_ordering(n, rp.ctypes.data, ci.ctypes.data, perm.ctypes.data)
    if rc != 0:
        raise MpeigError("rcm_ordering failed")
    return perm


def sparse_cholesky(A: Operator, precision: int = LOWER, perm="rcm") -> Operator:
    """Sparse Cholesky f_T = Pi L^-T L^-1 Pi^T (Preconditioner<T>::build(CsrMatrix,
    prec[, perm]), precond.hpp:55-77).  perm: "rcm" (the reference's default
    ordering), None (identity: the system was permuted upstream), or an array.
    `A` must be a csr_matrix() operator.  `.shift` = shift_applied(), `.factor_nnz`."""
    keep = ()
    if isinstance(perm, str):
        if perm != "rcm":
            raise ConfigError(f"unknown ordering {perm!r}")
        h = _mk(A.ctx, A.ctx.lib.mpeig_precond_sparse_chol, A.h, precision, 0, None)
    elif perm is None:
        h = _mk(A.ctx, A.ctx.lib.mpeig_precond_sparse_chol, A.h, precision, 1, None)
    else:
        p = np.ascontiguousarray(perm, dtype=np.int64)
        if p.size != A.n:
            raise DimensionMismatch("sparse_cholesky: bad permutation length")
        keep = (p,)
        h = _mk(A.ctx, A.ctx.lib.mpeig_precond_sparse_chol, A.h, precision, 2, p.ctypes.data)
    op = Operator(A.ctx, h, A.n, "sparse_chol", keep=(A,) + keep)
    op.shift = float(A.ctx.lib.mpeig_precond_shift(h))
    op.factor_nnz = int(A.ctx.lib.mpeig_precond_factor_nnz(h))
    return op


def solve_csr(row_ptr, col_idx, vals, cfg: "SolverConfig", ctx: Context = None,
              want_X: bool = True, history: bool = True) -> "EigResult":
    """The reference's stock sparse driver solve(CsrMatrix, cfg) (drivers.hpp:183-210)
    through mpeig_solve_csr: one RCM permutation of the system, the sparse Cholesky
    preconditioner at the variant's precision on the permuted system (identity
    ordering), the solve, and the eigenvectors returned in the original row order."""
    torch = _torch()
    ctx = ctx or default_context()
    rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(col_idx, dtype=np.int64)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    n = rp.size - 1
    k = cfg.k
    theta, resid = np.zeros(k), np.zeros(k)
    res = L.Result()
    res.theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    res.residual_norms = resid.ctypes.data_as(C.POINTER(C.c_double))
    X = None
    if want_X:
        X = torch.empty((k, n), dtype=torch.float64, device=f"cuda:{ctx.device}")
        res.X, res.ldx = C.c_void_p(X.data_ptr()), n
    hist = _History()
    shift = C.c_double(0.0)
    c = cfg.to_c()
    ctx.check(ctx.lib.mpeig_solve_csr(ctx.h, n, rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                      C.byref(c), hist.cb if history else L.SINK(), None,
                                      C.byref(res), C.byref(shift)))
    r = EigResult(theta, X.cpu().numpy() if X is not None else None, resid,
                  res.iterations_lower, res.iterations_working, hist.records, bool(res.converged),
                  _timings(res.timings), res.a_norm_estimate)
    r.precond_shift = shift.value
    return r


def build_precision_for(variant: str) -> int:
    """drivers.hpp:113-116."""
    return WORKING if variant == "dlobpcg-dchol" else LOWER


# ----------------------------------------------------------------- solvers


class _History:
    def __init__(self):
        self.records: List[IterationRecord] = []

        def sink(user, rec_p):
            r = rec_p.contents
            m = r.m
            self.records.append(IterationRecord(
                int(r.stage), [r.ritz_values[j] for j in range(m)],
                [r.residual_norms[j] for j in range(m)], int(r.n_converged),
                int(r.w_columns_dropped), bool(r.basis_rotation_fallback), time.perf_counter()))
        self.cb = L.SINK(sink)


def _timings(t: L.Timings) -> StageTimings:
    return StageTimings(t.factorize, t.precond_apply, t.orthogonalize, t.projected_eig, t.total)


def spectral_norm_estimate(A: Operator, sketch_rows: int = 8, seed: int = 0) -> float:
    out = C.c_double()
    A.ctx.check(A.ctx.lib.mpeig_spectral_norm_estimate(A.ctx.h, A.h, sketch_rows,
                                                       seed & 0xFFFFFFFFFFFFFFFF, C.byref(out)))
    return out.value


def solve(A: Operator, cfg: SolverConfig, T: Operator = None, want_X: bool = True,
          history: bool = True) -> EigResult:
    """solve() (drivers.hpp:158-181) with a Jacobi f_T at the variant's precision."""
    torch = _torch()
    ctx = A.ctx
    if T is None:
        T = jacobi(A, build_precision_for(cfg.variant))
    k = cfg.k
    theta = np.zeros(k)
    resid = np.zeros(k)
    X = None
    res = L.Result()
    res.theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    res.residual_norms = resid.ctypes.data_as(C.POINTER(C.c_double))
    if want_X:
        X = torch.empty((k, A.n), dtype=torch.float64, device=f"cuda:{ctx.device}")
        res.X, res.ldx = C.c_void_p(X.data_ptr()), A.n
    hist = _History()
    c = cfg.to_c()
    ctx.check(ctx.lib.mpeig_solve(ctx.h, A.h, T.h, C.byref(c),
                                  hist.cb if history else L.SINK(), None, C.byref(res)))
    return EigResult(theta, X, resid, res.iterations_lower, res.iterations_working,
                     hist.records, bool(res.converged), _timings(res.timings),
                     res.a_norm_estimate)


def solve_prepared(A: Operator, cfg: SolverConfig, X0raw, omega, omega_fro: float = 0.0,
                   T: Operator = None, X_out=None, history: bool = False) -> EigResult:
    """solve() from device-resident raw inputs (X0raw = gaussian_matrix(n, m, seed),
    omega = gaussian_matrix(n, sketch_rows, seed ^ 0x9e37...)): the benchmark's timed region."""
    ctx = A.ctx
    if T is None:
        T = jacobi(A, build_precision_for(cfg.variant))
    k = cfg.k
    theta, resid = np.zeros(k), np.zeros(k)
    res = L.Result()
    res.theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    res.residual_norms = resid.ctypes.data_as(C.POINTER(C.c_double))
    if X_out is not None:
        res.X, res.ldx = C.c_void_p(X_out.data_ptr()), X_out.shape[1]
    hist = _History()
    c = cfg.to_c()
    ctx.check(ctx.lib.mpeig_solve_prepared(
        ctx.h, A.h, T.h, C.byref(c), C.c_void_p(X0raw.data_ptr()), X0raw.shape[1],
        C.c_void_p(omega.data_ptr()), omega.shape[1], omega_fro,
        hist.cb if history else L.SINK(), None, C.byref(res)))
    return EigResult(theta, X_out, resid, res.iterations_lower, res.iterations_working,
                     hist.records, bool(res.converged), _timings(res.timings),
                     res.a_norm_estimate)


class profile:
    """Context manager: per-kernel-class CUDA-event timing inside the library."""

    def __enter__(self):
        lib = L.load()
        lib.mpeig_profile_reset()
        lib.mpeig_profile_enable(1)
        return self

    def __exit__(self, *exc):
        L.load().mpeig_profile_enable(0)

    @staticmethod
    def report() -> dict:
        lib = L.load()
        buf = C.create_string_buffer(8192)
        lib.mpeig_profile_names(buf, 8192)
        out = {}
        for name in buf.value.decode().split():
            cnt, ms, b, f = C.c_int64(), C.c_double(), C.c_double(), C.c_double()
            if lib.mpeig_profile_query(name.encode(), C.byref(cnt), C.byref(ms), C.byref(b),
                                       C.byref(f)) == 0:
                out[name] = {"count": cnt.value, "ms": ms.value, "bytes": b.value, "flops": f.value}
        return out


def run_variant(A: Operator, X0, cfg: SolverConfig, a_norm_est: float, T: Operator = None,
                want_X: bool = True) -> EigResult:
    """detail::run_variant (drivers.hpp:57-111) on an explicit fp64 device start block."""
    torch = _torch()
    ctx = A.ctx
    if T is None:
        T = jacobi(A, build_precision_for(cfg.variant))
    k = cfg.k
    theta, resid = np.zeros(k), np.zeros(k)
    X = None
    res = L.Result()
    res.theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    res.residual_norms = resid.ctypes.data_as(C.POINTER(C.c_double))
    if want_X:
        X = torch.empty((k, A.n), dtype=torch.float64, device=f"cuda:{ctx.device}")
        res.X, res.ldx = C.c_void_p(X.data_ptr()), A.n
    hist = _History()
    c = cfg.to_c()
    ctx.check(ctx.lib.mpeig_run_variant(ctx.h, A.h, T.h, C.byref(c), C.c_void_p(X0.data_ptr()),
                                        X0.shape[1], a_norm_est, hist.cb, None, C.byref(res)))
    return EigResult(theta, X, resid, res.iterations_lower, res.iterations_working, hist.records,
                     bool(res.converged), _timings(res.timings), res.a_norm_estimate)


def mixed_lobpcg(A: Operator, X0, cfg: SolverConfig, T: Operator = None) -> EigResult:
    """mixed_lobpcg (drivers.hpp:122-152): forces MPLOBPCG_schol; f_T built at LOWER
    precision (fp32 Jacobi unless T is given, e.g. dense_cholesky(A, LOWER))."""
    cfg = SolverConfig(**{**cfg.__dict__, "variant": "mplobpcg-schol"})
    est = spectral_norm_estimate(A, cfg.sketch_rows, cfg.seed ^ 0x9E3779B97F4A7C15)
    return run_variant(A, X0, cfg, est, T if T is not None else jacobi(A, LOWER))


def lobpcg_stage(A: Operator, n: int, X0, cfg: SolverConfig, T: Operator, a_norm_est: float,
                 opt: StageOptions, history: list = None, tim: StageTimings = None) -> StageOutcome:
    """lobpcg_stage<T> (eigensolvers.hpp:195-321); dtype of X0 picks T (f64/f32)."""
    torch = _torch()
    ctx = A.ctx
    m, ldx = X0.shape
    Xo = torch.empty((m, n), dtype=X0.dtype, device=X0.device)
    theta, resid = np.zeros(m), np.zeros(m)
    out = L.StageOut(C.c_void_p(Xo.data_ptr()), n, theta.ctypes.data_as(C.POINTER(C.c_double)),
                     resid.ctypes.data_as(C.POINTER(C.c_double)), 0, 0)
    hist = _History()
    t = L.Timings()
    c = cfg.to_c()
    o = L.StageOpts(opt.tol, int(opt.use_mixed_qr), int(opt.stagnation_exit), opt.tag)
    fn = ctx.lib.mpeig_lobpcg_stage_f64 if X0.dtype == torch.float64 else ctx.lib.mpeig_lobpcg_stage_f32
    rc = fn(ctx.h, A.h, n, C.c_void_p(X0.data_ptr()), ldx, m, C.byref(c), T.h, a_norm_est,
            C.byref(o), hist.cb, None, C.byref(out), C.byref(t))
    if history is not None:
        history.extend(hist.records)
    if tim is not None:
        tim.precond_apply += t.precond_apply
        tim.orthogonalize += t.orthogonalize
        tim.projected_eig += t.projected_eig
    ctx.check(rc)
    return StageOutcome(Xo, theta, resid, int(out.iterations), bool(out.converged))


def pinvit(A: Operator, n: int, X0, cfg: SolverConfig, T: Operator, a_norm_est: float = 0.0):
    """pinvit<double> (eigensolvers.hpp:326-390), preconditioner as an operator."""
    torch = _torch()
    ctx = A.ctx
    m, ldx = X0.shape
    k = cfg.k
    theta, resid = np.zeros(k), np.zeros(k)
    X = torch.empty((k, n), dtype=torch.float64, device=X0.device)
    res = L.Result()
    res.theta = theta.ctypes.data_as(C.POINTER(C.c_double))
    res.residual_norms = resid.ctypes.data_as(C.POINTER(C.c_double))
    res.X, res.ldx = C.c_void_p(X.data_ptr()), n
    hist = _History()
    c = cfg.to_c()
    ctx.check(ctx.lib.mpeig_pinvit_f64(ctx.h, A.h, n, C.c_void_p(X0.data_ptr()), ldx, m,
                                       C.byref(c), T.h, a_norm_est, hist.cb, None, C.byref(res)))
    return EigResult(theta, X, resid, 0, res.iterations_working, hist.records,
                     bool(res.converged), _timings(res.timings), res.a_norm_estimate)


def converged_count(a_norm_est: float, xnorm, theta, rnorm, tol: float) -> int:
    """converged_count (eigensolvers.hpp:25-43) on precomputed column norms."""
    n_c = 0
    for j in range(len(theta)):
        if rnorm[j] <= tol * (a_norm_est + abs(theta[j])) * xnorm[j]:
            n_c += 1
        else:
            break
    return n_c


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """gaussian_matrix<double> (dense_matrix.hpp:144-161), bit-exact stream."""
    out = np.zeros((rows, cols), order="F")
    rc = L.load().mpeig_gaussian_matrix_host(rows, cols, seed & 0xFFFFFFFFFFFFFFFF, out.ctypes.data)
    if rc != 0:
        raise MpeigError("gaussian_matrix failed")
    return out


# ------------------------------------------------- device <-> host helpers

def to_device(A: np.ndarray, dtype=None, device: int = 0):
    """n x c host block -> (c, n) contiguous CUDA tensor (column-major block)."""
    torch = _torch()
    A = np.asarray(A)
    if A.ndim == 1:
        A = A[:, None]
    t = torch.from_numpy(np.ascontiguousarray(A.T))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(f"cuda:{device}")


def to_host(X, n: int = None) -> np.ndarray:
    """(c, ld) CUDA tensor -> n x c numpy (Fortran order)."""
    a = X.detach().cpu().numpy()
    if n is not None:
        a = a[:, :n]
    return np.asfortranarray(a.T)
