"""CPU oracles -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this package, and only as the checker (or the
timed reference arm), never as the product path.

Two checkers share the C ABI in ``mp_oracle.h``:

* ``Oracle("ref")``  -> ``oracle/_ref/libmpeig_ref.so``: the unmodified reference
  library (``/root/reference/proj``) compiled here by ``oracle/Makefile`` and
  driven through its own ``lobpcg_stage`` / ``BlockOperator`` API
  (``oracle/ref_harness.cpp``).
* ``Oracle("port")`` -> ``oracle/liboracle.so``: ``oracle/mp_oracle.c``, a plain-C
  restatement of the reference algorithm, pinned against the reference in
  ``tests/test_oracle.py`` and against the reference's golden vectors.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {"ref": os.path.join(HERE, "_ref", "libmpeig_ref.so"),
        "port": os.path.join(HERE, "liboracle.so")}
PREFIX = {"ref": "mpref_", "port": "mporc_"}

VARIANTS = {"dlobpcg-dchol": 0, "dlobpcg-schol": 1, "mplobpcg-schol": 2, "pinvit": 3}
PROB_LAP3D, PROB_LAP2D, PROB_CSR, PROB_DENSE = 0, 1, 2, 3

ERRORS = {0: "OK", 1: "DimensionMismatch", 2: "ConfigError", 3: "NotPositiveDefinite",
          4: "SingularTriangular", 5: "RankDeficient", 6: "RankCollapse",
          7: "NoConvergence", 8: "OverflowError", 99: "Error"}


class MpProblem(C.Structure):
    _fields_ = [("kind", C.c_int32), ("nx", C.c_int64), ("ny", C.c_int64),
                ("nz", C.c_int64), ("n", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int64)),
                ("vals", C.POINTER(C.c_double)), ("dense", C.POINTER(C.c_double))]


class MpCfg(C.Structure):
    _fields_ = [("k", C.c_int64), ("block", C.c_int64), ("maxit", C.c_int64),
                ("tol", C.c_double), ("lower_tol", C.c_double), ("seed", C.c_uint64),
                ("sketch_rows", C.c_int64), ("x0", C.POINTER(C.c_double))]


class MpResult(C.Structure):
    _fields_ = [("converged", C.c_int32), ("status", C.c_int32),
                ("iters_lower", C.c_int64), ("iters_working", C.c_int64),
                ("a_norm_est", C.c_double),
                ("theta", C.POINTER(C.c_double)), ("resid", C.POINTER(C.c_double)),
                ("X", C.POINTER(C.c_double)),
                ("hist_cap", C.c_int64), ("hist_len", C.c_int64),
                ("hist_stage", C.POINTER(C.c_int32)), ("hist_nc", C.POINTER(C.c_int64)),
                ("hist_dropped", C.POINTER(C.c_int64)),
                ("hist_fallback", C.POINTER(C.c_int32)),
                ("hist_ritz", C.POINTER(C.c_double)), ("hist_resid", C.POINTER(C.c_double)),
                ("t_total", C.c_double), ("t_setup", C.c_double), ("t_stage1", C.c_double),
                ("msg", C.c_char * 256)]


def _ptr(a, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


@dataclass
class Problem:
    """A symmetric test matrix: 3-D 7-pt / 2-D 5-pt Laplacian, CSR or dense."""
    kind: int
    nx: int = 0
    ny: int = 0
    nz: int = 0
    n: int = 0
    row_ptr: np.ndarray | None = None
    col_idx: np.ndarray | None = None
    vals: np.ndarray | None = None
    dense: np.ndarray | None = None  # column-major (Fortran) n x n

    @staticmethod
    def lap3d(nx, ny=None, nz=None):
        ny = nx if ny is None else ny
        nz = nx if nz is None else nz
        return Problem(PROB_LAP3D, nx, ny, nz, n=nx * ny * nz)

    @staticmethod
    def lap2d(nx, ny=None):
        ny = nx if ny is None else ny
        return Problem(PROB_LAP2D, nx, ny, 1, n=nx * ny)

    @staticmethod
    def csr(row_ptr, col_idx, vals):
        return Problem(PROB_CSR, n=len(row_ptr) - 1,
                       row_ptr=np.ascontiguousarray(row_ptr, np.int64),
                       col_idx=np.ascontiguousarray(col_idx, np.int64),
                       vals=np.ascontiguousarray(vals, np.float64))

    @staticmethod
    def dense_matrix(A):
        A = np.asfortranarray(A, dtype=np.float64)
        return Problem(PROB_DENSE, n=A.shape[0], dense=A)

    def to_c(self):
        p = MpProblem()
        p.kind, p.nx, p.ny, p.nz, p.n = self.kind, self.nx, self.ny, self.nz, self.n
        p.row_ptr = _ptr(self.row_ptr, C.c_int64)
        p.col_idx = _ptr(self.col_idx, C.c_int64)
        p.vals = _ptr(self.vals, C.c_double)
        p.dense = self.dense.ctypes.data_as(C.POINTER(C.c_double)) if self.dense is not None else None
        return p


@dataclass
class SolveResult:
    status: int
    msg: str
    converged: bool
    iters_lower: int
    iters_working: int
    a_norm_est: float
    theta: np.ndarray
    resid: np.ndarray
    X: np.ndarray | None
    hist_stage: np.ndarray
    hist_nc: np.ndarray
    hist_dropped: np.ndarray
    hist_fallback: np.ndarray
    hist_ritz: np.ndarray
    hist_resid: np.ndarray
    t_total: float
    t_setup: float
    extra: dict = field(default_factory=dict)

    @property
    def iterations(self):
        return self.iters_lower + self.iters_working


class Oracle:
    def __init__(self, which: str = "port"):
        path = LIBS[which]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (make -C oracle)")
        self.which = which
        self.lib = C.CDLL(path)
        self.p = PREFIX[which]

    def fn(self, name):
        return getattr(self.lib, self.p + name)

    # ------------------------------------------------------------------ solve
    def solve(self, prob: Problem, variant: str, k: int, block: int = 0, maxit: int = 2000,
              tol: float = 1e-12, lower_tol: float = 5e-6, seed: int = 0,
              sketch_rows: int = 8, want_X: bool = False, hist_cap: int | None = None,
              native: bool = False, x0: np.ndarray | None = None):
        """native=True (reference library only, dense problems): the reference's
        stock solve(DenseMatrix, cfg) with its own Cholesky preconditioner
        (drivers.hpp:158-181) instead of the Jacobi-callback harness.
        x0 (n x m, Jacobi-callback harness only): the start block before
        orthonormal_q, in place of gaussian_matrix(n, m, seed)."""
        m = block if block else (3 * k + 1) // 2
        if x0 is not None:
            if native:
                raise ValueError("x0 override needs the callback harness (native=False)")
            x0 = np.asfortranarray(x0, dtype=np.float64)
            if x0.shape != (prob.n, m):
                raise ValueError(f"x0 must be {prob.n} x {m}")
        cfg = MpCfg(k, block, maxit, tol, lower_tol, seed, sketch_rows, _ptr(x0, C.c_double))
        hc = hist_cap if hist_cap is not None else 2 * maxit + 4
        theta = np.zeros(k)
        resid = np.zeros(k)
        X = np.zeros((prob.n, k), order="F") if want_X else None
        hs = np.zeros(hc, np.int32)
        hn = np.zeros(hc, np.int64)
        hd = np.zeros(hc, np.int64)
        hf = np.zeros(hc, np.int32)
        hr = np.zeros((hc, m))
        hq = np.zeros((hc, m))
        r = MpResult()
        r.theta, r.resid = _ptr(theta, C.c_double), _ptr(resid, C.c_double)
        r.X = X.ctypes.data_as(C.POINTER(C.c_double)) if X is not None else None
        r.hist_cap = hc
        r.hist_stage, r.hist_nc = _ptr(hs, C.c_int32), _ptr(hn, C.c_int64)
        r.hist_dropped, r.hist_fallback = _ptr(hd, C.c_int64), _ptr(hf, C.c_int32)
        r.hist_ritz, r.hist_resid = _ptr(hr, C.c_double), _ptr(hq, C.c_double)
        pc = prob.to_c()
        f = self.fn("solve_native" if native else "solve")
        f.argtypes = [C.POINTER(MpProblem), C.c_int, C.POINTER(MpCfg), C.POINTER(MpResult)]
        f(C.byref(pc), VARIANTS[variant], C.byref(cfg), C.byref(r))
        L = min(r.hist_len, hc)
        return SolveResult(r.status, r.msg.decode(errors="replace"), bool(r.converged),
                           r.iters_lower, r.iters_working, r.a_norm_est, theta, resid, X,
                           hs[:L], hn[:L], hd[:L], hf[:L], hr[:L], hq[:L], r.t_total,
                           r.t_setup, {"t_stage1": r.t_stage1})

    # ---------------------------------------------------------- unit kernels
    def pcg64(self, seed, count):
        out = np.zeros(count, np.uint64)
        f = self.fn("pcg64_u64")
        f.argtypes = [C.c_uint64, C.c_int64, C.POINTER(C.c_uint64)]
        f(seed, count, _ptr(out, C.c_uint64))
        return out

    def gaussian(self, rows, cols, seed):
        out = np.zeros((rows, cols), order="F")
        f = self.fn("gaussian")
        f.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_void_p]
        f(rows, cols, seed, out.ctypes.data)
        return out

    def norm_estimate(self, prob, sketch_rows=8, seed=0 ^ 0x9E3779B97F4A7C15):
        f = self.fn("norm_estimate")
        f.argtypes = [C.POINTER(MpProblem), C.c_int64, C.c_uint64]
        f.restype = C.c_double
        pc = prob.to_c()
        return f(C.byref(pc), sketch_rows, seed)

    def _qr(self, name, A, dtype=np.float64):
        A = np.asfortranarray(A, dtype=dtype)
        n, m = A.shape
        Q = np.zeros((n, m), dtype, order="F")
        R = np.zeros((m, m), dtype, order="F")
        f = self.fn(name)
        f.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        st = f(n, m, A.ctypes.data, Q.ctypes.data, R.ctypes.data)
        return st, Q, R

    def householder_qr(self, A):
        return self._qr("householder_qr", A)

    def householder_qr_f32(self, A):
        return self._qr("householder_qr_f32", A, np.float32)

    def mixed_qr(self, A):
        return self._qr("mixed_qr", A)

    def cholesky_qr(self, A):
        return self._qr("cholesky_qr", A)

    def small_herm_eig(self, M):
        M = np.asfortranarray(M, dtype=np.float64)
        n = M.shape[0]
        vals = np.zeros(n)
        vecs = np.zeros((n, n), order="F")
        f = self.fn("small_herm_eig")
        f.argtypes = [C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
        st = f(n, M.ctypes.data, vals.ctypes.data, vecs.ctypes.data)
        return st, vals, vecs

    def hl_update(self, S, Cm, m):
        S = np.asfortranarray(S, dtype=np.float64)
        Cm = np.asfortranarray(Cm, dtype=np.float64)
        n, s = S.shape
        p = min(m, s - m)
        X = np.zeros((n, m), order="F")
        P = np.zeros((n, p), order="F")
        cpv = np.zeros((s, p), order="F")
        fb = C.c_int32(0)
        f = self.fn("hl_update")
        f.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_void_p, C.c_void_p, C.POINTER(C.c_int32)]
        st = f(n, s, m, S.ctypes.data, Cm.ctypes.data, X.ctypes.data, P.ctypes.data,
               cpv.ctypes.data, C.byref(fb))
        return st, X, P, cpv, fb.value

    def project_out(self, B, W, passes):
        B = np.asfortranarray(B, dtype=np.float64)
        W = np.array(W, dtype=np.float64, order="F", copy=True)
        f = self.fn("project_out")
        f.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p, C.c_int]
        f(B.shape[0], B.shape[1], W.shape[1], B.ctypes.data, W.ctypes.data, passes)
        return W

    def ortho_dropping(self, W, tol):
        W = np.asfortranarray(W, dtype=np.float64)
        Q = np.zeros_like(W, order="F")
        f = self.fn("ortho_dropping")
        f.argtypes = [C.c_int64, C.c_int64, C.c_void_p, C.c_double, C.c_void_p]
        f.restype = C.c_int64
        kept = f(W.shape[0], W.shape[1], W.ctypes.data, tol, Q.ctypes.data)
        return np.asfortranarray(Q[:, :kept])

    def apply_op(self, prob, X):
        X = np.asfortranarray(X, dtype=np.float64)
        Y = np.zeros_like(X, order="F")
        f = self.fn("apply_op")
        f.argtypes = [C.POINTER(MpProblem), C.c_int64, C.c_void_p, C.c_void_p]
        pc = prob.to_c()
        f(C.byref(pc), X.shape[1], X.ctypes.data, Y.ctypes.data)
        return Y

    def converged_count(self, a_norm_est, X, theta, R, tol):
        X = np.asfortranarray(X, dtype=np.float64)
        R = np.asfortranarray(R, dtype=np.float64)
        theta = np.ascontiguousarray(theta, dtype=np.float64)
        f = self.fn("converged_count")
        f.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p,
                      C.c_double]
        f.restype = C.c_int64
        return f(X.shape[0], X.shape[1], a_norm_est, X.ctypes.data, theta.ctypes.data,
                 R.ctypes.data, tol)


def available(which: str) -> bool:
    return os.path.exists(LIBS[which])
