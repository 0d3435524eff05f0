"""Row-sharded (multi-GPU) path, SURVEY.md §8(e).

CPU: the sharding arithmetic that must agree across ranks (start-block row
slices bit for bit, slab partition) and the N > 1 launcher plumbing (NCCL id
creation + broadcast over a world-size-2 gloo group).
GPU: the sharded solver with ranks as threads of one process (host-staged
exchanges, rank-ordered sums) against the single-GPU solve and the global
operator.  NCCL itself needs one GPU per rank and is exercised by the
multi-GPU bench (bench.py --shard).
"""
import os
import threading

import numpy as np
import pytest

import paper_2302_12528_b200 as mp


@pytest.mark.parametrize("n,cols,parts", [(97, 5, 3), (1000, 3, 4), (64, 2, 1), (33, 7, 5)])
def test_gaussian_row_slices_bitwise(n, cols, parts):
    """Each rank draws exactly its rows of gaussian_matrix (dense_matrix.hpp:144-161)."""
    G = mp.gaussian_matrix(n, cols, 11)
    bounds = np.linspace(0, n, parts + 1).astype(int)
    got = np.vstack([mp.gaussian_matrix_rows(n, cols, 11, a, b - a)
                     for a, b in zip(bounds[:-1], bounds[1:])])
    assert np.array_equal(got, G)


def test_slab_partition():
    for nz, p in [(32, 3), (8, 8), (256, 8), (7, 2)]:
        sl = mp.slab_partition(nz, p)
        assert sum(n for _, n in sl) == nz and sl[0][0] == 0
        assert all(a + n == b for (a, n), (b, _) in zip(sl, sl[1:]))
        assert max(n for _, n in sl) - min(n for _, n in sl) <= 1


def _gloo_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    uid = mp.broadcast_unique_id(rank)
    out.put((rank, uid, mp.slab_partition(32, world)[rank]))
    dist.barrier()
    dist.destroy_process_group()


def test_nccl_id_broadcast_world2():
    """The N > 1 launcher path: rank 0's NCCL id reaches rank 1 (gloo, CPU)."""
    import socket

    import torch.multiprocessing as tmp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (u, sl)) for r, u, sl in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert len(res[0][0]) == 128 and res[0][0] == res[1][0]
    assert res[0][1] == (0, 16) and res[1][1] == (16, 16)


def _gloo_inputs_worker(rank, world, port, out):
    """Each rank builds its share of a sharded run's inputs the way bench.py does
    (slab, start block and sketch rows), gathers them over gloo, and rank 0
    compares with the single-process draw; the timings reduce by max."""
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    nx, ny, nz, m, seed = 6, 5, 11, 4, 7
    z0, nzl = mp.slab_partition(nz, world)[rank]
    n_glob, row0, n = nx * ny * nz, nx * ny * z0, nx * ny * nzl
    X0 = mp.gaussian_matrix_rows(n_glob, m, seed, row0, n)
    Om = mp.gaussian_matrix_rows(n_glob, 3, seed ^ 0x9E3779B97F4A7C15, row0, n)
    sizes = [None] * world
    dist.all_gather_object(sizes, (row0, n))
    parts = [None] * world
    dist.all_gather_object(parts, (X0, Om))
    t = torch.tensor([0.1 * (rank + 1), 0.2 * (world - rank)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        ok_rows = all(a + b == c for (a, b), (c, _) in zip(sizes, sizes[1:])) and \
            sizes[-1][0] + sizes[-1][1] == n_glob
        X = np.vstack([p[0] for p in parts])
        O = np.vstack([p[1] for p in parts])
        out.put((ok_rows, np.array_equal(X, mp.gaussian_matrix(n_glob, m, seed)),
                 np.array_equal(O, mp.gaussian_matrix(n_glob, 3, seed ^ 0x9E3779B97F4A7C15)),
                 t.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_inputs_gloo(world):
    """The N > 1 host plumbing on CPU ranks (gloo): the slab partition covers the
    rows in rank order, every rank's start block / sketch rows are bitwise the
    global draw's, and the per-rank times reduce by max."""
    import socket

    import torch.multiprocessing as tmp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gloo_inputs_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    ok_rows, ok_x, ok_o, t = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok_rows and ok_x and ok_o
    assert t == [0.1 * world, 0.2 * world]


# ------------------------------------------------------------------ GPU


def _run_ranks(nranks, dims, fn, ks_seed=None):
    """fn(rank, ctx, op_slab) on `nranks` threads sharing one HostGroup
    (ks_seed: the slab of cfg5's -Laplacian + V instead of the Laplacian)."""
    import torch
    nx, ny, nz = dims
    group = mp.HostGroup(nranks)
    slabs = mp.slab_partition(nz, nranks)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            ctx = mp.Context(0, stream=torch.cuda.Stream())
            ctx.attach_host(group, r)
            z0, nl = slabs[r]
            A = (mp.laplace3d_slab(nx, ny, nz, z0, nl, ctx=ctx) if ks_seed is None else
                 mp.ks_hamiltonian_slab(nx, ny, nz, z0, nl, seed=ks_seed, ctx=ctx))
            out[r] = fn(r, ctx, A)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,dims", [(2, (9, 8, 13)), (3, (9, 8, 13)), (2, (33, 5, 140)),
                                          (2, (64, 64, 1100))])
def test_sharded_stencil_apply_bitwise(gpu, nranks, dims):
    """Halo exchange + slab apply == the global apply, bit for bit (the
    vectorised per-point kernel and, on the large slabs, the z-marching one)."""
    n = int(np.prod(dims))
    X = np.asfortranarray(np.random.default_rng(3).standard_normal((n, 4)))
    Y = mp.to_host(gpu.laplace3d(*dims).apply(mp.to_device(X)))
    sl = mp.slab_partition(dims[2], nranks)
    plane = dims[0] * dims[1]

    def fn(r, ctx, A):
        z0, nl = sl[r]
        Xl = np.asfortranarray(X[z0 * plane:(z0 + nl) * plane])
        return mp.to_host(A.apply(mp.to_device(Xl)))

    parts = _run_ranks(nranks, dims, fn)
    assert np.array_equal(np.vstack(parts), Y)


@pytest.mark.gpu
@pytest.mark.parametrize("nranks,dims", [(2, (9, 8, 13)), (3, (16, 8, 21))])
def test_sharded_ks_apply_bitwise(gpu, nranks, dims):
    """The row-sharded variable-diagonal (cfg5) operator == its global apply,
    bit for bit, with the overlapped halo exchange."""
    n = int(np.prod(dims))
    X = np.asfortranarray(np.random.default_rng(4).standard_normal((n, 3)))
    Y = mp.to_host(gpu.ks_hamiltonian(*dims, seed=2).apply(mp.to_device(X)))
    sl = mp.slab_partition(dims[2], nranks)
    plane = dims[0] * dims[1]

    def fn(r, ctx, A):
        z0, nl = sl[r]
        Xl = np.asfortranarray(X[z0 * plane:(z0 + nl) * plane])
        return mp.to_host(A.apply(mp.to_device(Xl)))

    parts = _run_ranks(nranks, dims, fn, ks_seed=2)
    assert np.array_equal(np.vstack(parts), Y)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dlobpcg-dchol", "mplobpcg-schol"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_solve_matches_single_gpu(gpu, nranks, variant):
    """Row-sharded solve == single-GPU solve: theta to 1e-10, residual contract
    on the gathered X, iteration count within the rounding band."""
    dims = (10, 11, 12)
    cfg = mp.SolverConfig(k=5, tol=1e-10, maxit=1500, variant=variant)
    prec = mp.WORKING if variant == "dlobpcg-dchol" else mp.LOWER
    A1 = gpu.laplace3d(*dims)
    r1 = gpu.solve(A1, cfg, T=gpu.jacobi(A1, prec))

    def fn(r, ctx, A):
        res = mp.solve(A, cfg, T=mp.jacobi(A, prec))
        return res, mp.to_host(res.X)

    outs = _run_ranks(nranks, dims, fn)
    th0 = outs[0][0].theta
    for res, _ in outs:  # every rank holds the same replicated results
        assert np.array_equal(res.theta, th0)
        assert (res.iterations_lower, res.iterations_working) == (
            outs[0][0].iterations_lower, outs[0][0].iterations_working)
    res = outs[0][0]
    assert res.converged
    assert np.abs(res.theta - r1.theta).max() <= 1e-10 * np.abs(r1.theta).max()
    tot1 = r1.iterations_lower + r1.iterations_working
    tot = res.iterations_lower + res.iterations_working
    assert abs(tot - tot1) <= max(2, int(0.1 * tot1)), (tot, tot1)
    X = np.vstack([x for _, x in outs])
    assert np.linalg.norm(X.T @ X - np.eye(cfg.k)) < 1e-10
    AX = mp.to_host(A1.apply(mp.to_device(np.asfortranarray(X))))
    rn = np.linalg.norm(AX - X * res.theta, axis=0)
    assert np.all(rn <= 10 * cfg.tol * (res.a_norm_estimate + res.theta))


@pytest.mark.gpu
@pytest.mark.parametrize("transport", ["nccl", "host"])
def test_one_rank_sharded_path(gpu, transport):
    """A 1-rank communicator runs the full sharded code path (stacked TSQR,
    allreduced Grams / norms, status max, halo exchange with no neighbours)
    on one GPU; with NCCL this drives the real ncclAllReduce / AllGather /
    grouped send-recv calls.  Same answer as the unsharded solve."""
    import torch
    dims = (10, 11, 12)
    cfg = mp.SolverConfig(k=5, tol=1e-10, maxit=1500, variant="mplobpcg-schol")
    A1 = gpu.laplace3d(*dims)
    r1 = gpu.solve(A1, cfg, T=gpu.jacobi(A1, mp.LOWER))
    ctx = mp.Context(0, stream=torch.cuda.Stream())
    if transport == "nccl":
        ctx.attach_nccl(0, 1, mp.nccl_unique_id())
    else:
        group = mp.HostGroup(1)
        ctx.attach_host(group, 0)
    A = mp.laplace3d_slab(*dims, 0, dims[2], ctx=ctx)
    res = mp.solve(A, cfg, T=mp.jacobi(A, mp.LOWER))
    assert res.converged
    assert np.abs(res.theta - r1.theta).max() <= 1e-10 * np.abs(r1.theta).max()
    tot1 = r1.iterations_lower + r1.iterations_working
    tot = res.iterations_lower + res.iterations_working
    assert abs(tot - tot1) <= max(2, int(0.1 * tot1)), (tot, tot1)


# ------------------------------------------------------- sharded CSR (ghost rows)


def _row_blocks(n, nranks, seed=0):
    """Uneven contiguous row blocks in rank order (each within +-25 % of n / nranks:
    the sharded QR needs every block at least as tall as the basis is wide)."""
    rng = np.random.default_rng(seed)
    even = n / nranks
    cuts = [int(round(even * (r + 1) + rng.uniform(-0.25, 0.25) * even)) for r in range(nranks - 1)]
    b = np.concatenate([[0], cuts, [n]])
    return [(int(a), int(c - a)) for a, c in zip(b[:-1], b[1:])]


def _csr_block(rp, ci, v, r0, nl):
    lo, hi = rp[r0], rp[r0 + nl]
    return rp[r0:r0 + nl + 1] - lo, ci[lo:hi], v[lo:hi]


def _run_csr_ranks(nranks, n, rp, ci, v, blocks, fn):
    """fn(rank, ctx, op_rows) on `nranks` thread-ranks sharing one HostGroup."""
    import torch
    group = mp.HostGroup(nranks)
    out, errs = [None] * nranks, []

    def work(r):
        try:
            ctx = mp.Context(0, stream=torch.cuda.Stream())
            ctx.attach_host(group, r)
            r0, nl = blocks[r]
            A = mp.csr_rows(n, r0, *_csr_block(rp, ci, v, r0, nl), ctx=ctx)
            out[r] = fn(r, ctx, A)
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    return out


def _long_range_csr(nx, ny, extra, seed):
    """5-pt Laplacian plus `extra` random symmetric long-range couplings: ghost
    rows from non-neighbouring ranks as well as the row-block neighbours."""
    from problems import lap_csr
    rp, ci, v = lap_csr(nx, ny)
    n = nx * ny
    rows = [dict(zip(ci[rp[i]:rp[i + 1]].tolist(), v[rp[i]:rp[i + 1]].tolist())) for i in range(n)]
    rng = np.random.default_rng(seed)
    for _ in range(extra):
        i, j = (int(t) for t in rng.integers(0, n, 2))
        if i != j:
            w = -0.25 * rng.random()
            rows[i][j] = rows[i].get(j, 0.0) + w
            rows[j][i] = rows[j].get(i, 0.0) + w
            rows[i][i] += 0.5
            rows[j][j] += 0.5
    rp2, ci2, v2 = [0], [], []
    for d in rows:
        for c in sorted(d):
            ci2.append(c)
            v2.append(d[c])
        rp2.append(len(ci2))
    return np.array(rp2, np.int64), np.array(ci2, np.int64), np.array(v2)


@pytest.mark.gpu
@pytest.mark.parametrize("nranks", [2, 3, 4])
@pytest.mark.parametrize("prec", ["working", "lower"])
def test_sharded_csr_apply_bitwise(gpu, nranks, prec):
    """Row-block CSR with ghost-row exchange (any peer, uneven blocks, rows with
    and without ghost entries) == the global spmv_block apply, bit for bit."""
    import torch
    nx, ny = 23, 19
    n = nx * ny
    rp, ci, v = _long_range_csr(nx, ny, 60, 7)
    dt, pr = (np.float64, mp.WORKING) if prec == "working" else (np.float32, mp.LOWER)
    X = np.asfortranarray(np.random.default_rng(5).standard_normal((n, 7)).astype(dt))
    Ag = gpu.csr_matrix(rp, ci, v)
    Y = mp.to_host(Ag.apply(mp.to_device(X), precision=pr))
    blocks = _row_blocks(n, nranks, seed=nranks)

    def fn(r, ctx, A):
        r0, nl = blocks[r]
        Xl = mp.to_device(np.asfortranarray(X[r0:r0 + nl]))
        out = A.apply(Xl, precision=pr)
        torch.cuda.synchronize()
        return mp.to_host(out)

    parts = _run_csr_ranks(nranks, n, rp, ci, v, blocks, fn)
    assert np.array_equal(np.vstack(parts), Y)


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["dlobpcg-dchol", "mplobpcg-schol"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_sharded_csr_solve_matches_single_gpu(gpu, nranks, variant):
    """cfg2's family (2-D 5-pt Laplacian, here as CSR) row-sharded over thread
    ranks with ghost-row exchange: same answer as the single-GPU solve."""
    from problems import lap_csr
    nx, ny = 26, 21
    n = nx * ny
    rp, ci, v = lap_csr(nx, ny)
    cfg = mp.SolverConfig(k=5, tol=1e-10, maxit=2000, variant=variant)
    prec = mp.WORKING if variant == "dlobpcg-dchol" else mp.LOWER
    A1 = gpu.csr_matrix(rp, ci, v)
    r1 = gpu.solve(A1, cfg, T=gpu.jacobi(A1, prec))
    blocks = _row_blocks(n, nranks, seed=11)

    def fn(r, ctx, A):
        res = mp.solve(A, cfg, T=mp.jacobi(A, prec))
        return res, mp.to_host(res.X)

    outs = _run_csr_ranks(nranks, n, rp, ci, v, blocks, fn)
    res = outs[0][0]
    for rr, _ in outs:
        assert np.array_equal(rr.theta, res.theta)
    assert res.converged
    assert np.abs(res.theta - r1.theta).max() <= 1e-10 * np.abs(r1.theta).max()
    tot1 = r1.iterations_lower + r1.iterations_working
    tot = res.iterations_lower + res.iterations_working
    assert abs(tot - tot1) <= max(2, int(0.1 * tot1)), (tot, tot1)
    X = np.vstack([x for _, x in outs])
    assert np.linalg.norm(X.T @ X - np.eye(cfg.k)) < 1e-10


@pytest.mark.gpu
def test_csr_rows_partition_errors(gpu):
    """Row blocks out of rank order are refused on every rank."""
    from problems import lap_csr
    rp, ci, v = lap_csr(8, 8)
    n = 64
    with pytest.raises(Exception):
        _run_csr_ranks(2, n, rp, ci, v, [(32, 32), (0, 32)], lambda r, ctx, A: None)


@pytest.mark.gpu
def test_csr_rows_invalid_block_raises_on_every_rank(gpu):
    """A rank whose block is invalid (column out of range) makes every rank raise
    after the partition exchange -- nobody is left waiting in a collective."""
    import torch
    from problems import lap_csr
    rp, ci, v = lap_csr(8, 8)
    n = 64
    group = mp.HostGroup(2)
    errs = [None, None]

    def work(r):
        try:
            ctx = mp.Context(0, stream=torch.cuda.Stream())
            ctx.attach_host(group, r)
            r0, nl = (0, 32) if r == 0 else (32, 32)
            brp, bci, bv = _csr_block(rp, ci, v, r0, nl)
            if r == 1:
                bci = bci.copy()
                bci[-1] = n + 5
            mp.csr_rows(n, r0, brp, bci, bv, ctx=ctx)
        except Exception as e:
            errs[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert all(not t.is_alive() for t in th)
    assert all(isinstance(e, mp.MpeigError) for e in errs), errs
