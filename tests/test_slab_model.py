"""CPU (gloo, world_size 2 and 4) model of the slab decomposition the CUDA path runs
(csrc/plan.cu arena_slab_*, csrc/poisson_pow2.cuh Layout / rowB / rowC).

Each process plays one rank: it keeps the rank's workspaces B and C as flat
row buffers laid out exactly like the device ones (chunked, j-blocked rows of
ncp complex), does the per-axis transforms with numpy on those rows, and moves
whole chunks with torch.distributed.all_to_all_single — the same contiguous
chunks the grouped ncclSend/ncclRecv move.  The gathered u must equal the CPU
oracle's.  This checks the decomposition, the chunk geometry and the exchange
order without GPUs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _ilog2(x):
    return int(x).bit_length() - 1


class Layout:
    """Mirror of poisson_pow2.cuh Layout (JB = min(ARENA_JBLOCK = 64, nj))."""

    def __init__(self, ni, nj):
        self.ni, self.nj = ni, nj
        self.nis, self.njs = _ilog2(ni), _ilog2(nj)
        self.jbs = _ilog2(min(64, nj))

    def lrow(self, c, il, jl):
        jb = 1 << self.jbs
        return (c << (self.nis + self.njs)) + (((jl >> self.jbs) * self.ni + il) << self.jbs) + (jl & (jb - 1))

    def rowB(self, il, j):
        return self.lrow(j >> self.njs, il, j & (self.nj - 1))

    def rowC(self, i, jl):
        return self.lrow(i >> self.nis, i & (self.ni - 1), jl)


def _rank_main(rank, world, port, n, f, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = world
    ni = nj = n // P
    nc = n // 2 + 1
    ncp = (nc + 7) // 8 * 8
    gB, gC = Layout(ni, n // P), Layout(n // P, nj)
    B = np.zeros((ni * n, ncp), dtype=np.complex128)
    C = np.zeros((n * nj, ncp), dtype=np.complex128)
    fs = f[rank * ni:(rank + 1) * ni]
    # K1: r2c along k, rows (il, j) -> rowB
    for il in range(ni):
        spec = np.fft.rfft(fs[il], axis=1)  # (j, nc)
        for j in range(n):
            B[gB.rowB(il, j), :nc] = spec[j]
    # K2: forward FFT along j
    for il in range(ni):
        rows = [gB.rowB(il, j) for j in range(n)]
        B[rows, :nc] = np.fft.fft(B[rows, :nc], axis=0)
    # all-to-all #1: chunk d of B -> rank d's C chunk `rank`
    send = torch.from_numpy(B.view(np.float64).copy().ravel())
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    C[:] = recv.numpy().view(np.complex128).reshape(C.shape)
    # K3: forward along i, Poisson symbol (fft_solver.cpp:66-79), backward along i
    sf = lambda k: k if k <= n // 2 else k - n  # noqa: E731
    ki = np.array([sf(i) for i in range(n)], dtype=np.float64)
    scale, four_pi2 = 1.0 / (float(n) * n * n), 4.0 * np.pi * np.pi
    for jl in range(nj):
        j = rank * nj + jl
        rows = [gC.rowC(i, jl) for i in range(n)]
        X = np.fft.fft(C[rows, :nc], axis=0)
        k2 = ki[:, None] ** 2 + float(sf(j)) ** 2 + np.arange(nc, dtype=np.float64)[None, :] ** 2
        with np.errstate(divide="ignore"):
            X *= np.where(k2 == 0.0, 0.0, scale / (four_pi2 * k2))
        C[rows, :nc] = np.fft.ifft(X, axis=0) * n
    # all-to-all #2 (reverse)
    send = torch.from_numpy(C.view(np.float64).copy().ravel())
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send)
    B[:] = recv.numpy().view(np.complex128).reshape(B.shape)
    # K4: backward along j;  K5: c2r along k (imaginary parts of DC / Nyquist ignored)
    us = np.empty((ni, n, n))
    for il in range(ni):
        rows = [gB.rowB(il, j) for j in range(n)]
        Y = np.fft.ifft(B[rows, :nc], axis=0) * n
        us[il] = np.fft.irfft(Y, n=n, axis=1) * n
    gathered = [torch.empty(ni * n * n, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(gathered, torch.from_numpy(us.ravel().copy()))
    if rank == 0:
        out.copy_(torch.cat(gathered))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,world", [(16, 2), (32, 4)])
def test_slab_decomposition_gloo(n, world):
    import oracle

    f = np.random.default_rng(n * world).uniform(-1, 1, (n, n, n))
    out = torch.zeros(n ** 3, dtype=torch.float64).share_memory_()
    mp.spawn(_rank_main, args=(world, _free_port(), n, f, out), nprocs=world, join=True)
    u = out.numpy().reshape(n, n, n)
    ref = oracle.poisson_solve(f)
    assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref)


def test_layout_chunks_are_contiguous_and_disjoint():
    """Chunk d of B (j in rank d's range) and chunk r of C (i in rank r's range)
    are the contiguous row ranges [d*ni*nj, (d+1)*ni*nj) the exchanges move."""
    for n, P in ((16, 2), (64, 8), (1024, 8), (2048, 4)):
        ni = nj = n // P
        gB = Layout(ni, n // P)
        for d in range(P):
            rows = {gB.rowB(il, j) for il in range(0, ni, max(1, ni // 8)) for j in range(d * nj, (d + 1) * nj)}
            assert min(rows) >= d * ni * nj and max(rows) < (d + 1) * ni * nj
        # same in-chunk position on both sides of the exchange
        gC = Layout(n // P, nj)
        r, d = P - 1, 0
        for il in (0, ni - 1):
            for jl in (0, nj - 1):
                b = gB.rowB(il, d * nj + jl) - d * ni * nj
                c = gC.rowC(r * ni + il, jl) - r * ni * nj
                assert b == c


# ---------------------------------------------------------------- chunked exchange
def _substeps(n, P, forward, S=4):
    """The sub-step ranges the slab's chunked COPY exchange uses (plan.cu slab_solve_chunked)."""
    ni = nj = n // P
    JB = min(64, nj)
    if forward:
        cf = min(S, ni)
        return [(k * ni // cf, (k + 1) * ni // cf) for k in range(cf)]
    nb = nj // JB
    cb = min(S, nb)
    return [((k * nb // cb) * JB, ((k + 1) * nb // cb) * JB) for k in range(cb)]


@pytest.mark.parametrize("n,P", [(16, 2), (64, 4), (256, 8), (1024, 8), (1024, 2), (2048, 4)])
def test_exchange_pieces_cover_chunk_once(n, P):
    """arena_slab_exchange_pieces (the rows each sub-step moves) tiles a chunk exactly once,
    and sub-step k forward holds only rows K1+K2 wrote for its i planes, backward only rows
    K3 wrote for its j lines — so gating sub-step k on those kernels is sufficient."""
    import paper_1408_6497_b200 as arena

    ni = nj = n // P
    g = Layout(ni, nj)
    for forward in (True, False):
        seen = np.zeros(ni * nj, dtype=np.int32)
        for lo, hi in _substeps(n, P, forward):
            pcs = arena.slab_exchange_pieces(n, P, forward, lo, hi)
            rows = np.concatenate([np.arange(a, a + c) for a, c in pcs])
            seen[rows] += 1
            # invert the in-chunk row -> (il, jl)
            jb = 1 << g.jbs
            blk, within = rows // jb, rows % jb
            il, jl = blk % ni, (blk // ni) * jb + within
            if forward:
                assert il.min() >= lo and il.max() < hi
            else:
                assert jl.min() >= lo and jl.max() < hi
        assert (seen == 1).all()


def _rank_main_chunked(rank, world, port, n, f, out, pieces_fwd, pieces_bwd):
    """The slab solve with the chunked exchange: K1+K2 per i-plane sub-range, each followed by
    that sub-step's all-to-all of the piece rows; K3 per j-block sub-range, each followed by
    the reverse sub-step.  Rows outside a sub-step's pieces must not be needed by it."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    P = world
    ni = nj = n // P
    nc = n // 2 + 1
    ncp = (nc + 7) // 8 * 8
    gB, gC = Layout(ni, n // P), Layout(n // P, nj)
    B = np.full((ni * n, ncp), np.nan, dtype=np.complex128)  # NaN: a row read before it arrives poisons u
    C = np.full((n * nj, ncp), np.nan, dtype=np.complex128)
    chunk = ni * nj
    fs = f[rank * ni:(rank + 1) * ni]

    def exchange(src, dst, pcs):
        rows = np.concatenate([np.arange(a, a + c) for a, c in pcs])
        send = np.concatenate([src[d * chunk + rows] for d in range(P)])
        recv = torch.empty(send.size * 2, dtype=torch.float64)
        dist.all_to_all_single(recv, torch.from_numpy(send.view(np.float64).ravel().copy()))
        got = recv.numpy().view(np.complex128).reshape(P, rows.size, ncp)
        for r in range(P):
            dst[r * chunk + rows] = got[r]

    for (lo, hi), pcs in zip(_substeps(n, P, True), pieces_fwd):
        for il in range(lo, hi):
            spec = np.fft.rfft(fs[il], axis=1)
            rws = [gB.rowB(il, j) for j in range(n)]
            B[rws, :nc] = np.fft.fft(spec, axis=0)
            B[rws, nc:] = 0
        exchange(B, C, pcs)
    sf = lambda k: k if k <= n // 2 else k - n  # noqa: E731
    ki = np.array([sf(i) for i in range(n)], dtype=np.float64)
    scale, four_pi2 = 1.0 / (float(n) * n * n), 4.0 * np.pi * np.pi
    for (lo, hi), pcs in zip(_substeps(n, P, False), pieces_bwd):
        for jl in range(lo, hi):
            j = rank * nj + jl
            rows = [gC.rowC(i, jl) for i in range(n)]
            X = np.fft.fft(C[rows, :nc], axis=0)
            k2 = ki[:, None] ** 2 + float(sf(j)) ** 2 + np.arange(nc, dtype=np.float64)[None, :] ** 2
            with np.errstate(divide="ignore"):
                X *= np.where(k2 == 0.0, 0.0, scale / (four_pi2 * k2))
            C[rows, :nc] = np.fft.ifft(X, axis=0) * n
        exchange(C, B, pcs)
    us = np.empty((ni, n, n))
    for il in range(ni):
        rows = [gB.rowB(il, j) for j in range(n)]
        Y = np.fft.ifft(B[rows, :nc], axis=0) * n
        us[il] = np.fft.irfft(Y, n=n, axis=1) * n
    gathered = [torch.empty(ni * n * n, dtype=torch.float64) for _ in range(P)]
    dist.all_gather(gathered, torch.from_numpy(us.ravel().copy()))
    if rank == 0:
        out.copy_(torch.cat(gathered))
    dist.destroy_process_group()


@pytest.mark.parametrize("n,world", [(16, 2), (32, 4)])
def test_slab_chunked_exchange_gloo(n, world):
    """World 2 / 4 with the chunked schedule and the pieces from the C ABI: equals the oracle."""
    import oracle
    import paper_1408_6497_b200 as arena

    pf = [arena.slab_exchange_pieces(n, world, True, lo, hi) for lo, hi in _substeps(n, world, True)]
    pb = [arena.slab_exchange_pieces(n, world, False, lo, hi) for lo, hi in _substeps(n, world, False)]
    assert len(pf) > 1
    f = np.random.default_rng(n + world).uniform(-1, 1, (n, n, n))
    out = torch.zeros(n ** 3, dtype=torch.float64).share_memory_()
    mp.spawn(_rank_main_chunked, args=(world, _free_port(), n, f, out, pf, pb), nprocs=world, join=True)
    u = out.numpy().reshape(n, n, n)
    ref = oracle.poisson_solve(f)
    assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref)
