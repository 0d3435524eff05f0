"""Kernel-level parity of the sm_100a path against the reference (via the oracle).

Bitwise for the elementwise / operator kernels (the reference's exact
operation order is reproduced), tolerance-level for reductions.
All calls go through the C ABI (libmpeig_b200.so).
"""
import ctypes as C

import numpy as np
import pytest

from oracle import Oracle, Problem, available

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def ref_or_port():
    return Oracle("ref") if available("ref") else Oracle("port")


def rand(n, m, seed, dtype=np.float64):
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((n, m)).astype(dtype))


@pytest.mark.parametrize("prob,mk", [
    (Problem.lap3d(8, 7, 6), lambda mp: mp.laplace3d(8, 7, 6)),
    (Problem.lap3d(5), lambda mp: mp.laplace3d(5)),
    (Problem.lap2d(9, 8), lambda mp: mp.laplace2d(9, 8)),
    (Problem.lap3d(37, 9, 70), lambda mp: mp.laplace3d(37, 9, 70)),
    # z-marching kernel (n >= 2^21): ragged last z-chunk, plane not a multiple of the CTA
    (Problem.lap3d(64, 50, 700), lambda mp: mp.laplace3d(64, 50, 700)),
    # y-marching 2-D kernel (n >= 2^20): row not a multiple of the CTA, ragged last chunk
    (Problem.lap2d(1030, 1021), lambda mp: mp.laplace2d(1030, 1021)),
])
def test_stencil_apply_bitwise(gpu, prob, mk):
    mp = gpu
    A = mk(mp)
    X = rand(prob.n, 5, 1)
    Y = mp.to_host(A.apply(mp.to_device(X)))
    Yr = ref_or_port().apply_op(prob, X)
    assert np.array_equal(Y, Yr), np.abs(Y - Yr).max()


def csr_of_lap2d(nx, ny):
    rp, ci, vv = [0], [], []
    for j in range(ny):
        for i in range(nx):
            p = i + nx * j
            ent = []
            if j > 0:
                ent.append((p - nx, -1.0))
            if i > 0:
                ent.append((p - 1, -1.0))
            ent.append((p, 4.0))
            if i + 1 < nx:
                ent.append((p + 1, -1.0))
            if j + 1 < ny:
                ent.append((p + nx, -1.0))
            for c, v in ent:
                ci.append(c)
                vv.append(v)
            rp.append(len(ci))
    return np.array(rp), np.array(ci), np.array(vv)


@pytest.mark.parametrize("dims", [(8, 7, 6), (37, 9, 70), (64, 50, 700)])
@pytest.mark.parametrize("precision", ["working", "lower"])
def test_ks_stencil_bitwise_vs_csr(gpu, dims, precision):
    """The variable-diagonal 7-pt stencil (H = -Laplacian + V, cfg5) equals the
    CSR SpMM of the same matrix bit for bit (both sum in CSR column order =
    the reference's spmv_block), in both precisions and every kernel form
    (scalar, vectorised, z-marching)."""
    mp = gpu
    from paper_2302_12528_b200.generators import ks_csr
    import torch
    H = mp.ks_hamiltonian(*dims, seed=3)
    Acsr = mp.csr_matrix(*ks_csr(*dims, seed=3))
    prec = mp.WORKING if precision == "working" else mp.LOWER
    dt = torch.float64 if precision == "working" else torch.float32
    X = torch.randn(5, H.n, dtype=dt, device="cuda")
    Y1 = H.apply(X, precision=prec)
    Y2 = Acsr.apply(X, precision=prec)
    assert torch.equal(Y1, Y2)


def test_csr_apply_bitwise(gpu):
    mp = gpu
    rp, ci, vv = csr_of_lap2d(11, 7)
    rng = np.random.default_rng(3)
    vv = vv * (1 + 0.1 * rng.random(len(vv)))  # non-trivial coefficients
    A = mp.csr_matrix(rp, ci, vv)
    X = rand(77, 4, 2)
    Y = mp.to_host(A.apply(mp.to_device(X)))
    Yr = ref_or_port().apply_op(Problem.csr(rp, ci, vv), X)
    assert np.array_equal(Y, Yr)


def test_dense_apply(gpu):
    mp = gpu
    M = rand(64, 64, 4)
    M = np.asfortranarray(M + M.T)
    A = mp.dense_matrix(M)
    X = rand(64, 3, 5)
    Y = mp.to_host(A.apply(mp.to_device(X)))
    assert np.allclose(Y, M @ X, rtol=0, atol=1e-12 * np.abs(M).sum())


@pytest.mark.parametrize("precision", [0, 1])
def test_residual_precond_bitwise(gpu, precision):
    """W = f_T(AX - X diag(theta)) bitwise; norms to 1e-15."""
    mp = gpu
    n, m = 4099, 11
    A = mp.laplace3d(n, 1, 1)  # only its diagonal (6) is used
    T = mp.jacobi(A, precision)
    X, AX = rand(n, m, 6), rand(n, m, 7)
    theta = np.random.default_rng(8).random(m)
    W = np.zeros((n, m), order="F")
    rn, xn = np.zeros(m), np.zeros(m)
    ctx = A.ctx
    Xd, AXd = mp.to_device(X), mp.to_device(AX)
    Wd = mp.to_device(W)
    ctx.check(ctx.lib.mpeig_residual_precond_f64(
        ctx.h, T.h, n, m, C.c_void_p(Xd.data_ptr()), n, C.c_void_p(AXd.data_ptr()), n,
        theta.ctypes.data, C.c_void_p(Wd.data_ptr()), n, rn.ctypes.data, xn.ctypes.data))
    W = mp.to_host(Wd)
    R = AX - X * theta[None, :]          # numpy: separate mul / sub, like the reference
    dinv = np.full(n, 1.0 / 6.0)
    if precision == 0:
        Wr = R * dinv[:, None]
    else:
        Wr = (R.astype(np.float32) * dinv.astype(np.float32)[:, None]).astype(np.float64)
    assert np.array_equal(W, Wr)
    assert np.allclose(rn, np.linalg.norm(R, axis=0), rtol=1e-14, atol=0)
    assert np.allclose(xn, np.linalg.norm(X, axis=0), rtol=1e-14, atol=0)


def test_residual_overflow_is_loud(gpu):
    mp = gpu
    n, m = 64, 2
    A = mp.laplace3d(4)
    T = mp.jacobi(A, 1)
    X = np.zeros((n, m), order="F")
    AX = np.zeros((n, m), order="F")
    AX[3, 1] = 1e300
    W = np.zeros((n, m), order="F")
    rn, xn = np.zeros(m), np.zeros(m)
    ctx = A.ctx
    Xd, AXd, Wd = mp.to_device(X), mp.to_device(AX), mp.to_device(W)
    rc = ctx.lib.mpeig_residual_precond_f64(
        ctx.h, T.h, n, m, C.c_void_p(Xd.data_ptr()), n, C.c_void_p(AXd.data_ptr()), n,
        np.zeros(m).ctypes.data, C.c_void_p(Wd.data_ptr()), n, rn.ctypes.data, xn.ctypes.data)
    assert rc == 8  # OverflowError


GRAM_SHAPES = [(100003, 48, 37), (1000, 144, 144), (31, 5, 7),
               # the m = 80 / 48 iteration's shapes: S^T AS 240^2, [X P]^T W 160 x 80,
               # W^T W 80^2 (80-wide DMMA tiles), 96 x 48, and a ragged 200 x 130
               (70001, 240, 240), (50000, 160, 80), (40003, 80, 80), (30000, 96, 48),
               (20011, 200, 130)]


@pytest.mark.parametrize("n,ka,kb", GRAM_SHAPES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_gram(gpu, n, ka, kb, dtype):
    """adjoint_matmul (dense_kernels.hpp:36-52) in both precisions against a
    float64 reference product; the error bound is the fp64 / fp32 dot-product
    bound sqrt(n) u ||a|| ||b|| per entry."""
    mp = gpu
    import torch
    npdt, tdt, u = ((np.float64, torch.float64, 2.0 ** -53) if dtype == "f64"
                    else (np.float32, torch.float32, 2.0 ** -24))
    A, B = rand(n, ka, 9, npdt), rand(n, kb, 10, npdt)
    ctx = mp.default_context()
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    Gd = torch.zeros((kb, ka), dtype=tdt, device="cuda")
    fn = ctx.lib.mpeig_gram_f64 if dtype == "f64" else ctx.lib.mpeig_gram_f32
    ctx.check(fn(ctx.h, n, ka, C.c_void_p(Ad.data_ptr()), n, kb, C.c_void_p(Bd.data_ptr()), n,
                 C.c_void_p(Gd.data_ptr())))
    G = Gd.cpu().numpy().T.astype(np.float64)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    Gr = A64.T @ B64
    scale = np.sqrt(np.outer((A64 * A64).sum(0), (B64 * B64).sum(0)))
    assert np.all(np.abs(G - Gr) <= 16 * u * np.sqrt(n) * scale + 1e-300)


@pytest.mark.parametrize("n,ka,kb", [(70001, 240, 240), (50000, 160, 80), (40003, 80, 80),
                                     (30000, 96, 48), (20011, 200, 130), (1000, 16, 16),
                                     (4099, 130, 7)])
def test_gram_f32_tensor_cores(gpu, n, ka, kb):
    """The binary32 Gram on tcgen05 (tc.cu, forced for every shape): the exact
    3-way bf16 split + fp32 accumulation matches the float64 product within the
    binary32 dot-product bound, and agrees with the SIMT FFMA kernel to the
    same level."""
    mp = gpu
    import torch
    A, B = rand(n, ka, 19, np.float32), rand(n, kb, 20, np.float32)
    A[::97, :] *= 1e-3  # dynamic range inside a column
    ctx = mp.default_context()
    Ad = torch.from_numpy(np.ascontiguousarray(A.T)).cuda()
    Bd = torch.from_numpy(np.ascontiguousarray(B.T)).cuda()
    out = {}
    for opt in (2, 0):
        assert ctx.lib.mpeig_set_process_option(b"gram_tc", opt) == 0
        try:
            Gd = torch.zeros((kb, ka), dtype=torch.float32, device="cuda")
            ctx.check(ctx.lib.mpeig_gram_f32(ctx.h, n, ka, C.c_void_p(Ad.data_ptr()), n, kb,
                                             C.c_void_p(Bd.data_ptr()), n, C.c_void_p(Gd.data_ptr())))
            out[opt] = Gd.cpu().numpy().T.astype(np.float64)
        finally:
            ctx.lib.mpeig_set_process_option(b"gram_tc", 1)
    A64, B64 = A.astype(np.float64), B.astype(np.float64)
    Gr = A64.T @ B64
    bound = 16 * 2.0 ** -24 * np.sqrt(n) * np.sqrt(np.outer((A64 * A64).sum(0), (B64 * B64).sum(0)))
    assert np.all(np.abs(out[2] - Gr) <= bound)
    assert np.all(np.abs(out[2] - out[0]) <= 2 * bound)
    # as accurate as the FFMA kernel (the tensor core's accumulation rounding
    # must not add up over the part products: ADR in tc.cu)
    sc = np.abs(A64).T @ np.abs(B64)
    e_tc, e_simt = np.max(np.abs(out[2] - Gr) / sc), np.max(np.abs(out[0] - Gr) / sc)
    assert e_tc <= 1.5 * e_simt + 2 * 2.0 ** -24, (e_tc, e_simt)


GEMM_SHAPES = [(50001, 96, 70), (40000, 240, 160), (30001, 160, 80), (20000, 80, 80),
               (10007, 144, 96), (5000, 48, 48)]


@pytest.mark.parametrize("n,k,c", GEMM_SHAPES)
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_gemm(gpu, n, k, c, dtype):
    """Y = Z - A C (matmul + subtract, dense_kernels.hpp:20-62), both precisions,
    every output-tile width class (16 .. 80 columns, several column tiles)."""
    mp = gpu
    import torch
    npdt, tdt, u = ((np.float64, torch.float64, 2.0 ** -53) if dtype == "f64"
                    else (np.float32, torch.float32, 2.0 ** -24))
    A, Cm, Z = rand(n, k, 11, npdt), rand(k, c, 12, npdt), rand(n, c, 13, npdt)
    ctx = mp.default_context()
    dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()  # noqa: E731
    Ad, Cd, Zd = dev(A), dev(Cm), dev(Z)
    fn = ctx.lib.mpeig_gemm_f64 if dtype == "f64" else ctx.lib.mpeig_gemm_f32
    ctx.check(fn(ctx.h, n, k, c, -1.0, C.c_void_p(Ad.data_ptr()), n, C.c_void_p(Cd.data_ptr()), k,
                 1.0, C.c_void_p(Zd.data_ptr()), n, C.c_void_p(Zd.data_ptr()), n))
    Y = Zd.cpu().numpy().T.astype(np.float64)
    Yr = Z.astype(np.float64) - A.astype(np.float64) @ Cm.astype(np.float64)
    bound = 4 * u * (np.abs(A).astype(np.float64) @ np.abs(Cm).astype(np.float64) + np.abs(Z)) * k
    assert np.all(np.abs(Y - Yr) <= bound)


@pytest.mark.parametrize("n,k,c", [(40000, 240, 160), (30001, 160, 80), (20000, 80, 80),
                                   (10007, 144, 96), (5000, 48, 48), (4099, 37, 13),
                                   (1000, 16, 200), (3001, 576, 384), (2000, 100, 256),
                                   (2500, 33, 257)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_gemm_f32_tensor_cores(gpu, n, k, c, beta):
    """The binary32 block update on tcgen05 (tc.cu, forced for every shape):
    exact 3-way bf16 split, fp32 accumulation; against float64 and against the
    SIMT FFMA kernel, with and without the beta Z term."""
    mp = gpu
    import torch
    A, Cm, Z = rand(n, k, 31, np.float32), rand(k, c, 32, np.float32), rand(n, c, 33, np.float32)
    ctx = mp.default_context()
    dev = lambda M: torch.from_numpy(np.ascontiguousarray(M.T)).cuda()  # noqa: E731
    Ad, Cd = dev(A), dev(Cm)
    out = {}
    for opt in (2, 0):
        assert ctx.lib.mpeig_set_process_option(b"gemm_tc", opt) == 0
        try:
            Zd = dev(Z)
            Yd = torch.zeros_like(Zd)
            ctx.check(ctx.lib.mpeig_gemm_f32(ctx.h, n, k, c, -1.0, C.c_void_p(Ad.data_ptr()), n,
                                             C.c_void_p(Cd.data_ptr()), k, beta,
                                             C.c_void_p(Zd.data_ptr()), n, C.c_void_p(Yd.data_ptr()), n))
            out[opt] = Yd.cpu().numpy().T.astype(np.float64)
        finally:
            ctx.lib.mpeig_set_process_option(b"gemm_tc", 1)
    Yr = beta * Z.astype(np.float64) - A.astype(np.float64) @ Cm.astype(np.float64)
    sc = np.abs(A).astype(np.float64) @ np.abs(Cm).astype(np.float64) + np.abs(Z)
    bound = 4 * 2.0 ** -24 * sc * k
    assert np.all(np.abs(out[2] - Yr) <= bound)
    assert np.all(np.abs(out[2] - out[0]) <= 2 * bound)
    e_tc, e_simt = np.max(np.abs(out[2] - Yr) / sc), np.max(np.abs(out[0] - Yr) / sc)
    assert e_tc <= 1.5 * e_simt + 2 * 2.0 ** -24, (e_tc, e_simt)


def test_gemm_inplace_wide_is_refused(gpu):
    """Y aliasing A: allowed only where one output column tile covers all of c
    (binary64 c <= 96; binary32 c <= 256 on the tensor-core path); wider, the
    column tiles would race, so the library refuses instead of
    returning wrong columns."""
    mp = gpu
    import torch
    n = 10000
    ctx = mp.default_context()
    for k in (97, 112):
        W = torch.randn(k, n, dtype=torch.float64, device="cuda")
        U = torch.eye(k, dtype=torch.float64, device="cuda")
        rc = ctx.lib.mpeig_gemm_f64(ctx.h, n, k, k, 1.0, C.c_void_p(W.data_ptr()), n,
                                    C.c_void_p(U.data_ptr()), k, 0.0, None, 0,
                                    C.c_void_p(W.data_ptr()), n)
        assert rc == 1  # DimensionMismatch
    # binary32 without the tensor-core path: the SIMT kernels tile c by 64
    W = torch.randn(80, n, dtype=torch.float32, device="cuda")
    U = torch.eye(80, dtype=torch.float32, device="cuda")
    assert ctx.lib.mpeig_set_process_option(b"gemm_tc", 0) == 0
    try:
        rc = ctx.lib.mpeig_gemm_f32(ctx.h, n, 80, 80, 1.0, C.c_void_p(W.data_ptr()), n,
                                    C.c_void_p(U.data_ptr()), 80, 0.0, None, 0,
                                    C.c_void_p(W.data_ptr()), n)
    finally:
        ctx.lib.mpeig_set_process_option(b"gemm_tc", 1)
    assert rc == 1


@pytest.mark.parametrize("dtype,k", [("f64", 80), ("f64", 96), ("f32", 80), ("f32", 192),
                                     ("f32", 256)])
def test_gemm_inplace_matches_out_of_place(gpu, dtype, k):
    """W <- W U in place (the CholQR V U^-1 step at m = 80 .. 256) is bitwise the
    out-of-place product: each CTA reads all k columns of its rows before its
    single column tile is written."""
    mp = gpu
    import torch
    n = 100004  # ld a multiple of 4: the aligned (in-place capable) kernels
    tdt = torch.float64 if dtype == "f64" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(k)
    W = torch.randn(k, n, dtype=tdt, device="cuda", generator=g)
    U = torch.randn(k, k, dtype=tdt, device="cuda", generator=g) / k ** 0.5
    ctx = mp.default_context()
    fn = ctx.lib.mpeig_gemm_f64 if dtype == "f64" else ctx.lib.mpeig_gemm_f32
    if dtype == "f32":
        assert ctx.lib.mpeig_set_process_option(b"gemm_tc", 2) == 0
    try:
        Y = torch.empty_like(W)
        ctx.check(fn(ctx.h, n, k, k, 1.0, C.c_void_p(W.data_ptr()), n, C.c_void_p(U.data_ptr()), k,
                     0.0, None, 0, C.c_void_p(Y.data_ptr()), n))
        ctx.check(fn(ctx.h, n, k, k, 1.0, C.c_void_p(W.data_ptr()), n, C.c_void_p(U.data_ptr()), k,
                     0.0, None, 0, C.c_void_p(W.data_ptr()), n))
    finally:
        ctx.lib.mpeig_set_process_option(b"gemm_tc", 1)
    torch.cuda.synchronize()
    assert torch.equal(W, Y)


def graded(n, m, kappa, seed):
    rng = np.random.default_rng(seed)
    Q1, _ = np.linalg.qr(rng.standard_normal((n, m)))
    Q2, _ = np.linalg.qr(rng.standard_normal((m, m)))
    s = kappa ** (-np.arange(m) / (m - 1))
    return np.asfortranarray((Q1 * s) @ Q2)


@pytest.mark.parametrize("kappa", [1e1, 1e3, 1e5, 1e7])
def test_mixed_qr_orthogonality(gpu, kappa):
    """acceptance criterion 6 (tests/acceptance.cpp:367-387): <= 100*200*u_h."""
    mp = gpu
    import torch
    n, m = 20000, 24
    A = graded(n, m, kappa, 17)
    Wd = mp.to_device(A)
    Rd = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    ctx = mp.default_context()
    ctx.check(ctx.lib.mpeig_mixed_qr_f64(ctx.h, n, m, C.c_void_p(Wd.data_ptr()), n,
                                         C.c_void_p(Rd.data_ptr())))
    Q, R = mp.to_host(Wd), mp.to_host(Rd)
    orth = np.linalg.norm(Q.T @ Q - np.eye(m))
    assert orth <= 100 * 200 * U
    assert np.all(np.diag(R) > 0)
    assert np.linalg.norm(Q @ R - A) <= 1e-12 * np.linalg.norm(A) * (1 + kappa * 1e-4)
    # same unique Q as the reference's Householder (to rounding x kappa)
    st, Qr, Rr = ref_or_port().mixed_qr(A)
    assert st == 0
    assert np.abs(Q - Qr).max() <= 1e-14 * kappa * 100


@pytest.mark.parametrize("n,m", [(3001, 16), (100, 7), (40000, 16), (5000, 32), (20000, 48),
                                 (9000, 64), (7000, 80), (3000, 96), (2000, 112),
                                 # long blocks: warp-leaf passes before the register TSQR
                                 (400000, 16), (330000, 48)])
def test_householder_qr_matches_reference(gpu, n, m):
    """TSQR tree shapes: one leaf, several tree levels, every register-tile width
    class and the shared-memory fallback (m > 96 in fp64)."""
    mp = gpu
    import torch
    A = rand(n, m, 21)
    Wd = mp.to_device(A)
    Rd = torch.zeros((m, m), dtype=torch.float64, device="cuda")
    ctx = mp.default_context()
    ctx.check(ctx.lib.mpeig_householder_qr_f64(ctx.h, n, m, C.c_void_p(Wd.data_ptr()), n,
                                               C.c_void_p(Rd.data_ptr())))
    Q, R = mp.to_host(Wd), mp.to_host(Rd)
    st, Qr, Rr = ref_or_port().householder_qr(A)
    assert np.abs(Q - Qr).max() < 1e-13 * max(1, m / 16)
    assert np.abs(R - Rr).max() < 1e-12 * np.abs(Rr).max()


def test_rank_deficient_drops(gpu):
    """orthonormal_q_dropping falls back to MGS with column dropping."""
    mp = gpu
    n = 500
    A = rand(n, 6, 22)
    A[:, 4] = A[:, 1] * 2.0  # exactly dependent
    A[:, 5] = 0.0            # vanished column
    Wd = mp.to_device(A)
    ctx = mp.default_context()
    kept = C.c_int64()
    ctx.check(ctx.lib.mpeig_orthonormal_q_dropping_f64(ctx.h, n, 6, C.c_void_p(Wd.data_ptr()), n,
                                                       1, C.byref(kept)))
    Qr = ref_or_port().ortho_dropping(A, np.sqrt(np.finfo(float).eps))
    assert kept.value == Qr.shape[1] == 4
    Q = mp.to_host(Wd)[:, :kept.value]
    assert np.linalg.norm(Q.T @ Q - np.eye(4)) < 1e-13
    assert np.abs(np.abs(Q) - np.abs(Qr)).max() < 1e-10


def test_project_out(gpu):
    mp = gpu
    n, b, w = 7000, 20, 8
    B, _ = np.linalg.qr(rand(n, b, 23))
    B = np.asfortranarray(B)
    W = rand(n, w, 24)
    Bd, Wd = mp.to_device(B), mp.to_device(W)
    ctx = mp.default_context()
    ctx.check(ctx.lib.mpeig_project_out_f64(ctx.h, n, b, C.c_void_p(Bd.data_ptr()), n, w,
                                            C.c_void_p(Wd.data_ptr()), n, 2))
    Y = mp.to_host(Wd)
    Yr = ref_or_port().project_out(B, W, 2)
    assert np.abs(Y - Yr).max() <= 1e-13
    assert np.abs(B.T @ Y).max() <= 1e-13


@pytest.mark.parametrize("s", [12, 48, 96])
@pytest.mark.parametrize("spectrum", ["random", "pairs"])
def test_small_eig(gpu, s, spectrum):
    """small_herm_eig (small_eig.hpp:92-218) against the reference's own values AND
    vectors (up to column sign): the Rayleigh-Ritz basis is what the block update
    consumes.  "pairs": eigenvalues in close pairs (relative split 1e-6), the
    near-degenerate clusters of the Laplacian's Ritz matrices."""
    mp = gpu
    import torch
    if spectrum == "random":
        M = rand(s, s, 25)
        M = M + M.T
    else:
        Q, _ = np.linalg.qr(rand(s, s, 26))
        lam = np.repeat(np.arange(1, s // 2 + 1, dtype=np.float64), 2)
        lam[1::2] *= 1 + 1e-6
        M = (Q * lam) @ Q.T
        M = 0.5 * (M + M.T)
    M = np.asfortranarray(M)
    Md = mp.to_device(M)
    vals = torch.zeros(s, dtype=torch.float64, device="cuda")
    vecs = torch.zeros((s, s), dtype=torch.float64, device="cuda")
    ctx = mp.default_context()
    ctx.check(ctx.lib.mpeig_small_eig_f64(ctx.h, s, C.c_void_p(Md.data_ptr()),
                                          C.c_void_p(vals.data_ptr()), C.c_void_p(vecs.data_ptr())))
    st, vr, Vr = ref_or_port().small_herm_eig(M)
    v = vals.cpu().numpy()
    scale = np.abs(vr).max()
    assert np.abs(v - vr).max() <= 1e-13 * scale
    V = mp.to_host(vecs)
    assert np.linalg.norm(M @ V - V * v) <= 1e-12 * scale
    gap = np.min(np.diff(vr)) / scale
    sign = np.sign(np.sum(V * Vr, axis=0))
    err = np.abs(V * sign - Vr).max()
    assert err <= 1e-13 / gap, (err, gap)


def test_hl_coeffs_match_reference(gpu):
    """hl_update (eigensolvers.hpp:148-174) rotation from identical C."""
    mp = gpu
    import torch
    n, s, m = 30, 12, 4
    S, _ = np.linalg.qr(rand(n, s, 44))
    H = rand(s, s, 45)
    G = H.T @ H
    st, vals, Cm = ref_or_port().small_herm_eig(G)
    st, Xr, Pr, cpv_r, fb_r = ref_or_port().hl_update(S, Cm, m)
    Cd = mp.to_device(Cm)
    coef = torch.zeros((2 * m, s), dtype=torch.float64, device="cuda")
    p, fb = C.c_int64(), C.c_int32()
    ctx = mp.default_context()
    ctx.check(ctx.lib.mpeig_hl_coeffs_f64(ctx.h, s, m, C.c_void_p(Cd.data_ptr()),
                                          C.c_void_p(coef.data_ptr()), C.byref(p), C.byref(fb)))
    cf = mp.to_host(coef)
    assert p.value == m and fb.value == fb_r == 0
    assert np.array_equal(cf[:, :m], Cm[:, :m])
    assert np.abs(cf[:, m:] - cpv_r).max() <= 1e-13


@pytest.mark.gpu
def test_default_context_orders_with_torch_default_stream(gpu):
    """A Context on torch's default stream runs on its own stream; each call
    must still wait for earlier default-stream work (a non-blocking H2D copy)
    and finish before later default-stream work (the D2H read)."""
    import torch
    A = gpu.laplace3d(256, 256, 128)
    n = A.n
    Xh = torch.from_numpy(np.random.default_rng(1).standard_normal((2, n))).pin_memory()
    Xd = Xh.to("cuda:0")
    torch.cuda.synchronize()
    ref = A.apply(Xd).cpu()
    for _ in range(3):
        xd = Xh.to("cuda:0", non_blocking=True)  # still in flight on the default stream
        got = A.apply(xd).cpu()
        assert torch.equal(got, ref)
