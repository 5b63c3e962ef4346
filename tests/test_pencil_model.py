"""CPU (gloo) model of the pencil decomposition the CUDA path runs
(csrc/plan.cu arena_pencil_*, csrc/pow2_launch.cuh pencil_phase_n,
csrc/poisson_pow2.cuh k_zfwd_pencil / k_zinv_pencil / Layout).

Each process plays rank (r, c) of a Pr x Pc grid and keeps its buffers as flat
row arrays laid out exactly like the device ones: R (K1 output, Pc k-chunks of
pitch kq, rows in Layout(ni, nj) order), Y (after the row exchange, chunk q =
column q's rows), B2 (K2 output, j re-chunked by n/Pr), C (after the column
exchange).  The exchanges are torch.distributed all_to_all_single calls on the
row / column sub-groups moving whole chunks — the same contiguous blocks the
grouped ncclSend/ncclRecv (or the peer stores) move.  The gathered u must equal
the CPU oracle's."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from test_slab_model import Layout


def pencil_kq(n, pc):
    """launchers.h pencil_kq: ceil(nc / Pc) rounded up to 8 (or 4, 2) keeping every chunk non-empty."""
    nc = n // 2 + 1
    w = (nc + pc - 1) // pc
    for q in (8, 4, 2):
        kq = (w + q - 1) // q * q
        if (pc - 1) * kq < nc:
            return kq
    return w


def _a2a(buf, group):
    send = torch.from_numpy(np.ascontiguousarray(buf).view(np.float64).ravel().copy())
    recv = torch.empty_like(send)
    dist.all_to_all_single(recv, send, group=group)
    return recv.numpy().view(np.complex128).reshape(buf.shape)


def _rank_main(rank, world, port, n, pr, pc, f, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = [dist.new_group([r * pc + q for q in range(pc)]) for r in range(pr)]
    cols = [dist.new_group([q * pc + c for q in range(pr)]) for c in range(pc)]
    r, c = rank // pc, rank % pc
    ni, nj, nj2 = n // pr, n // pc, n // pr
    nc, kq = n // 2 + 1, pencil_kq(n, pc)
    k0, kc = c * kq, min(kq, nc - c * kq)  # this rank's k chunk after the row exchange
    gz, gY, gB2, gC = Layout(ni, nj), Layout(ni, nj), Layout(ni, nj2), Layout(ni, nj2)
    blk = f[r * ni:(r + 1) * ni, c * nj:(c + 1) * nj]

    # K1: r2c along k, row (il, jl) -> k-chunk q at lrow(gz, 0, il, jl)
    R = np.zeros((pc, ni * nj, kq), dtype=np.complex128)
    for il in range(ni):
        for jl in range(nj):
            spec = np.fft.rfft(blk[il, jl])
            row = gz.lrow(0, il, jl)
            for q in range(pc):
                seg = spec[q * kq:(q + 1) * kq]
                R[q, row, :len(seg)] = seg
    Y = _a2a(R, rows[r])  # row exchange: chunk q -> rank (r, q), at chunk c

    # K2: y forward over all j for each (il, local k); output rows rowB(gB2, il, j)
    Yf = Y.reshape(pc * ni * nj, kq)
    B2 = np.zeros((pr * ni * nj2, kq), dtype=np.complex128)
    for il in range(ni):
        src = [gY.rowB(il, j) for j in range(n)]
        dst = [gB2.rowB(il, j) for j in range(n)]
        B2[dst, :kc] = np.fft.fft(Yf[src, :kc], axis=0)
    C = _a2a(B2.reshape(pr, ni * nj2, kq), cols[c]).reshape(pr * ni * nj2, kq)  # column exchange

    # K3: x forward * symbol (fft_solver.cpp:66-79) * x backward over all i
    sf = lambda k: k if k <= n // 2 else k - n  # noqa: E731
    ki = np.array([sf(i) for i in range(n)], dtype=np.float64)
    kk = np.arange(k0, k0 + kc, dtype=np.float64)
    for jl in range(nj2):
        j = r * nj2 + jl
        rows_i = [gC.rowC(i, jl) for i in range(n)]
        X = np.fft.fft(C[rows_i, :kc], axis=0)
        k2 = ki[:, None] ** 2 + float(sf(j)) ** 2 + kk[None, :] ** 2
        with np.errstate(divide="ignore"):
            X *= np.where(k2 == 0.0, 0.0, 1.0 / (n ** 3 * 4.0 * np.pi ** 2 * k2))
        C[rows_i, :kc] = np.fft.ifft(X, axis=0) * n

    # the reverse: column exchange, K4 y backward, row exchange, K5 c2r
    B2 = _a2a(C.reshape(pr, ni * nj2, kq), cols[c]).reshape(pr * ni * nj2, kq)
    Yb = np.zeros((pc * ni * nj, kq), dtype=np.complex128)
    for il in range(ni):
        src = [gB2.rowB(il, j) for j in range(n)]
        dst = [gY.rowB(il, j) for j in range(n)]
        Yb[dst, :kc] = np.fft.ifft(B2[src, :kc], axis=0) * n
    R = _a2a(Yb.reshape(pc, ni * nj, kq), rows[r])
    ub = np.empty((ni, nj, n))
    for il in range(ni):
        for jl in range(nj):
            row = gz.lrow(0, il, jl)
            spec = np.concatenate([R[q, row] for q in range(pc)])[:nc]
            ub[il, jl] = np.fft.irfft(spec, n=n) * n

    gathered = [torch.empty(ni * nj * n, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(gathered, torch.from_numpy(ub.ravel().copy()))
    if rank == 0:
        full = np.empty((n, n, n))
        for q, g in enumerate(gathered):
            rr, cc = q // pc, q % pc
            full[rr * ni:(rr + 1) * ni, cc * nj:(cc + 1) * nj] = g.numpy().reshape(ni, nj, n)
        out.copy_(torch.from_numpy(full.ravel()))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n,pr,pc", [(16, 2, 2), (16, 1, 2), (16, 2, 1), (32, 2, 2)])
def test_pencil_decomposition_gloo(n, pr, pc):
    import oracle

    f = np.random.default_rng(n * 10 + pr * 3 + pc).uniform(-1, 1, (n, n, n))
    out = torch.zeros(n ** 3, dtype=torch.float64).share_memory_()
    mp.spawn(_rank_main, args=(pr * pc, _free_port(), n, pr, pc, f, out), nprocs=pr * pc, join=True)
    u = out.numpy().reshape(n, n, n)
    ref = oracle.poisson_solve(f)
    assert np.linalg.norm(u - ref) <= 1e-12 * np.linalg.norm(ref)


def test_pencil_kq_properties():
    """pencil_kq (restating launchers.h): pinned values and, for every grid, a
    non-empty last chunk and full k coverage (tiny grids may leave the last
    column without k; the kernels then skip that rank's work)."""
    assert pencil_kq(2048, 4) == 264
    assert pencil_kq(16, 2) == 8
    assert pencil_kq(64, 4) == 10  # 8- and 4-aligned pitches would leave rank 3 empty
    for n in (64, 128, 1024, 2048):  # the device pencil path needs n >= 64
        for pc in (1, 2, 4, 8):
            kq, nc = pencil_kq(n, pc), n // 2 + 1
            assert nc <= pc * kq  # all k covered
            w = -(-nc // pc)
            if (pc - 1) * w < nc:  # a non-empty last chunk is possible: the pitch keeps it
                assert (pc - 1) * kq < nc
