"""Multi-rank paths.

* GPU (-m gpu): the slab-decomposed 2D schedule of the library run as P
  virtual ranks on one GPU (the same kernels, blocked layouts and column
  offsets as the NCCL path; the all-to-alls become device copies), and the
  NCCL path itself with a 1-rank communicator -- against the oracle.
* CPU (gloo, world_size 2): the decomposition the library implements
  (row slabs, blocked all-to-all, column slabs,
  filter column offsets, scales), written out with numpy block moves and the
  oracle's 1D transforms as the local steps, exchanged with
  torch.distributed.all_to_all over gloo, must equal the oracle's full
  pipeline.  This pins the index maps and the host-side schedule.
"""
import os
import socket

import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")


# ------------------------------------------------------------------ GPU
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0103001_b200 as b

    b.load_library()
    return b


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", [False, True])
@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("N,M", [(64, 64), (256, 512), (2048, 2048)])
def test_virtual_ranks_pipeline(P, N, M, exchange, monkeypatch):
    """Fused schedule (row kernels store / load the blocks of the other
    ranks' column slabs directly) and, with B200FFT_DIST_EXCHANGE=1, the
    all-to-all schedule (send slab -> exchange -> receive slab)."""
    if exchange:
        monkeypatch.setenv("B200FFT_DIST_EXCHANGE", "1")
    b = _lib()
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=500 + P, dtype=np.complex64).reshape(N, M)
    p = b.Plan((N, M))
    p.set_virtual_ranks(P)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(od.cpu().numpy(), oracle.gauss_pipeline(f, 0.1)) <= 1e-5
    F = torch.empty_like(fd)
    p.forward(fd, F)
    g = torch.empty_like(fd)
    p.inverse(fd, g)
    torch.cuda.synchronize()
    assert oracle.rel_l2(F.cpu().numpy(), oracle.fft2d(f)) <= 1e-5
    assert oracle.rel_l2(g.cpu().numpy(), oracle.ifft2d(f)) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("exchange", [False, True])
@pytest.mark.parametrize("P,N,M", [(2, 4096, 1024), (4, 8192, 256), (8, 4096, 2048)])
def test_virtual_ranks_fourstep_columns(P, N, M, exchange, monkeypatch):
    """Long columns (N >= 4096): the column step on each [N][M/P] slab as the
    three four-step column passes (N = 4096) or the one-pass k_colfilt
    (N = 8192), pass B applying g_N[k1 + 64 k2] * g_M[col_off + v], batch
    of two grids."""
    if exchange:
        monkeypatch.setenv("B200FFT_DIST_EXCHANGE", "1")
    b = _lib()
    f = fixtures.complex_input(2 * N * M, fixtures.UNIFORM, seed=60 + P, dtype=np.complex64).reshape(2, N, M)
    p = b.Plan((N, M), batch=2)
    p.set_virtual_ranks(P)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    # N = 8192: the column step is one k_colfilt launch per slab; 4096: the
    # three four-step column passes
    cols = 1 if N == 8192 else 3
    assert p.last_launch_count() == 2 * (P + cols * P + P)
    p.destroy()
    out = od.cpu().numpy()
    for i in range(2):
        assert oracle.rel_l2(out[i], oracle.gauss_pipeline(f[i], 0.1)) <= 1e-5


@pytest.mark.gpu
def test_virtual_ranks_c4_shape_real_input():
    b = _lib()
    N = 8192
    f = fixtures.complex_input(N * N, fixtures.UNIFORM, seed=4).reshape(N, N)
    p = b.Plan((N, N))
    p.set_virtual_ranks(8)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(od.cpu().numpy(), oracle.gauss_pipeline(f, 0.1)) <= 1e-5
    img = fixtures.sky_image(512, 512, seed=3, nsrc=50)
    q = b.Plan((512, 512), flags=b.IN_REAL_F32)
    q.set_virtual_ranks(4)
    o2 = torch.empty((512, 512), dtype=torch.complex64, device="cuda")
    q.filter_pipeline(torch.from_numpy(img).cuda(), o2, b.FILTER_IDEAL_LITERAL, 200.0)
    torch.cuda.synchronize()
    u = np.arange(512)[:, None]
    v = np.arange(512)[None, :]
    H = np.where((u - 256) ** 2 + (v - 256) ** 2 <= 200.0 ** 2, 0.0, 1.0)
    assert oracle.rel_l2(o2.cpu().numpy(), oracle.filter_pipeline(img.astype(complex), H)) <= 1e-5


def _sched_env(monkeypatch, sched, P):
    """fused: distributed transposes into peer slabs (default); exchange: the
    pack -> all-to-all -> unpack schedule (device copies for virtual ranks,
    ncclSend/ncclRecv with a communicator)."""
    if sched == "exchange":
        monkeypatch.setenv("B200FFT_P2P" if P == 1 else "B200FFT_DIST_EXCHANGE", "0" if P == 1 else "1")


@pytest.mark.gpu
@pytest.mark.parametrize("sched", ["fused", "exchange"])
@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("m,dtype", [(8, np.complex64), (16, np.complex64), (20, np.complex64),
                                     (22, np.complex64), (18, np.complex128)])
def test_virtual_ranks_four_step_1d(P, m, dtype, sched, monkeypatch):
    """The distributed four-step 1D schedule (3 transposes across the ranks,
    natural order) as P virtual ranks (P = 1: a 1-rank NCCL communicator);
    forward (1/N) and inverse against the oracle."""
    _sched_env(monkeypatch, sched, P)
    b = _lib()
    n = 1 << m
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=600 + m, dtype=dtype)
    prec = b.C64 if dtype == np.complex64 else b.C128
    p = b.Plan((n,), batch=1, precision=prec)
    if P > 1:
        p.set_virtual_ranks(P)
    else:
        p.set_comm(b.nccl_unique_id(), 1, 0)  # the NCCL exchange with one rank
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    zd = torch.empty_like(xd)
    p.forward(xd, yd)
    p.inverse(xd, zd)
    torch.cuda.synchronize()
    tol = 1e-5 if dtype == np.complex64 else 1e-12
    assert oracle.rel_l2(yd.cpu().numpy(), oracle.fft(x)) <= tol
    assert oracle.rel_l2(zd.cpu().numpy(), oracle.ifft(x)) <= tol
    p.destroy()


@pytest.mark.gpu
@pytest.mark.parametrize("sched", ["fused", "exchange"])
@pytest.mark.parametrize("P,m", [(2, 12), (4, 16), (8, 19)])
def test_virtual_ranks_four_step_transposed_output(P, m, sched, monkeypatch):
    """FFT_OUT_TRANSPOSED: rank r holds X[k2 + N2 k1] for its k2 block at
    local index (k2 - r N2/P) N1 + k1."""
    _sched_env(monkeypatch, sched, P)
    b = _lib()
    n = 1 << m
    N1, N2 = 1 << (m - m // 2), 1 << (m // 2)
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=700 + m)
    p = b.Plan((n,), batch=1, flags=b.OUT_TRANSPOSED)
    p.set_virtual_ranks(P)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    torch.cuda.synchronize()
    X = oracle.fft(x)
    # rank-major concatenation of [k2 local][k1] blocks == [k2][k1] overall
    expected = X.reshape(N1, N2).T.ravel()  # X[k2 + N2 k1] at k2 * N1 + k1
    assert oracle.rel_l2(yd.cpu().numpy(), expected) <= 1e-5
    p.destroy()


@pytest.mark.gpu
def test_virtual_ranks_c5_shape():
    """BASELINE configs[4] layout: N = 2^30 over 8 virtual ranks (32768 x
    32768 four-step, the fused distributed transposes): forward on seed 5 and
    inverse on the independent seed-105 input, each on 64 bins against the
    oracle's direct compensated sums."""
    b = _lib()
    n = 1 << 30
    x = np.empty(n, np.complex64)
    fixtures.complex_input(n, fixtures.NORMAL, seed=5, out=x)
    p = b.Plan((n,), batch=1)
    p.set_virtual_ranks(8)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    torch.cuda.synchronize()
    bins = np.concatenate([[0, 1, n // 2, n - 1], np.random.default_rng(55).integers(0, n, 60)])
    got = yd[torch.from_numpy(bins).cuda()].cpu().numpy()
    assert oracle.rel_l2(got, oracle.dft_bins(x, bins)) <= 1e-5
    fixtures.complex_input(n, fixtures.NORMAL, seed=105, out=x)
    xd.copy_(torch.from_numpy(x))
    p.inverse(xd, yd)
    torch.cuda.synchronize()
    bins = np.concatenate([[0, 1, n // 2, n - 1], np.random.default_rng(155).integers(0, n, 60)])
    got = yd[torch.from_numpy(bins).cuda()].cpu().numpy()
    assert oracle.rel_l2(got, oracle.dft_bins(x, bins, inverse=True)) <= 1e-5
    p.destroy()


@pytest.mark.gpu
@pytest.mark.parametrize("p2p", ["1", "0"])
def test_nccl_single_rank_communicator(p2p, monkeypatch):
    """The communicator data path with one rank: the fused peer-memory
    schedule (IPC handle exchange over NCCL, stream-ordered NCCL barriers) and,
    with B200FFT_P2P=0, the ncclSend/ncclRecv all-to-all schedule."""
    monkeypatch.setenv("B200FFT_P2P", p2p)
    b = _lib()
    N = M = 512
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=77).reshape(N, M)
    p = b.Plan((N, M), batch=1)
    p.set_comm(b.nccl_unique_id(), 1, 0)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    for _ in range(3):  # both receive phases and back
        p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    assert oracle.rel_l2(od.cpu().numpy(), oracle.gauss_pipeline(f, 0.1)) <= 1e-5
    F = torch.empty_like(fd)
    p.forward(fd, F)
    torch.cuda.synchronize()
    assert oracle.rel_l2(F.cpu().numpy(), oracle.fft2d(f)) <= 1e-5
    p.destroy()


# ------------------------------------------------------- CPU (gloo, 2 ranks)
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rows_blocked(a, SM):
    """k_rows' blocked store: slab [SN][M] -> blocks q of [SN][SM] (peer q's columns)."""
    SN, M = a.shape
    return np.ascontiguousarray(a.reshape(SN, M // SM, SM).transpose(1, 0, 2))  # [q][SN][SM]


def _unblock(blocks):
    """k_rows' blocked load: blocks [q][SN][SM] -> slab [SN][M]."""
    P, SN, SM = blocks.shape
    return np.ascontiguousarray(blocks.transpose(1, 0, 2).reshape(SN, P * SM))


def _a2a(dist, blocks):
    """All-to-all of blocks[q] -> rank q as point-to-point pairs (the library
    issues the same per-peer ncclSend/ncclRecv inside one NCCL group; gloo
    has no alltoall)."""
    send = torch.from_numpy(np.ascontiguousarray(blocks))
    recv = torch.empty_like(send)
    me = dist.get_rank()
    reqs = []
    for q in range(dist.get_world_size()):
        if q == me:
            recv[q].copy_(send[q])
        else:
            reqs.append(dist.isend(send[q].contiguous(), q))
            reqs.append(dist.irecv(recv[q], q))
    for r in reqs:
        r.wait()
    return recv.numpy()


def _worker(rank, world, port, N, M, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = world
        SN, SM = N // P, M // P
        f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=11, dtype=np.complex128).reshape(N, M)
        slab = f[rank * SN:(rank + 1) * SN]
        # 1. rows: unnormalised forward (M * the paper's 1/M DFT), blocked store
        rows = np.stack([oracle.fft(r) * M for r in slab])
        recv = _a2a(dist, _rows_blocked(rows, SM))  # [p][SN][SM] = column slab [N][SM]
        cs = recv.reshape(N, SM)
        # 2. columns: forward (1/N) -> * H(u, v + r SM) / M ... the library's
        #    combined scale H/(N M) on the unnormalised transforms
        H = oracle.gauss_filter(N, M, 0.1)[:, rank * SM:(rank + 1) * SM]
        colf = np.stack([oracle.fft(cs[:, j]) for j in range(SM)], axis=1)  # (1/N) sum
        colf *= H / M  # eq5's 1/N is in oracle.fft; the 2D-IDFT's 1/M here
        coli = np.stack([oracle.ifft(colf[:, j]) for j in range(SM)], axis=1)
        back = _a2a(dist, coli.reshape(P, SN, SM))  # blocks by source rank
        # 3. rows inverse (unscaled) from the blocked layout
        out = np.stack([oracle.ifft(r) for r in _unblock(back)])
        ref = oracle.gauss_pipeline(f, 0.1)[rank * SN:(rank + 1) * SN]
        q.put((rank, oracle.rel_l2(out, ref)))
    except Exception as exc:  # report instead of hanging the parent
        q.put((rank, f"error: {exc!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,M", [(16, 16), (64, 32)])
def test_gloo_two_rank_slab_schedule(N, M):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, M, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=60) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0] <= 1e-13 and res[1] <= 1e-13, res


def _unpack(recv, P):
    """[P][R][Cb] blocks by source rank -> [R][P*Cb] (the library's unpack_blocks)."""
    _, R, Cb = recv.shape
    return np.ascontiguousarray(recv.transpose(1, 0, 2).reshape(R, P * Cb))


def _worker_1d(rank, world, port, m, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P = world
        n = 1 << m
        N1, N2 = 1 << (m - m // 2), 1 << (m // 2)
        S1, S2 = N1 // P, N2 // P
        x = fixtures.complex_input(n, fixtures.NORMAL, seed=21, dtype=np.complex128)
        A = x[rank * n // P:(rank + 1) * n // P].reshape(S2, N1)  # rows n2 of x[n1 + N1 n2]
        # 1. pack = transpose; exchange blocks of [S1][S2]; unpack to [S1][N2]
        u = _unpack(_a2a(dist, A.T.copy().reshape(P, S1, S2)), P)
        # 2. (A) unnormalised FFT over n2, (T) twiddle W_n^{n1 k2}
        u = np.stack([oracle.fft(r) * N2 for r in u])
        n1 = rank * S1 + np.arange(S1)[:, None]
        k2 = np.arange(N2)[None, :]
        u = u * np.exp(-2j * np.pi * ((n1 * k2) % n) / n)
        # 3. pack, exchange, unpack to [S2][N1]; (B) FFT over n1 with 1/n overall
        z = _unpack(_a2a(dist, u.T.copy().reshape(P, S2, S1)), P)
        z = np.stack([oracle.fft(r) * N1 for r in z]) / n
        # 4. natural order: pack, exchange, unpack to [S1][N2] = X[r n/P, (r+1) n/P)
        out = _unpack(_a2a(dist, z.T.copy().reshape(P, S1, S2)), P).ravel()
        ref = oracle.fft(x)[rank * n // P:(rank + 1) * n // P]
        q.put((rank, oracle.rel_l2(out, ref)))
    except Exception as exc:
        q.put((rank, f"error: {exc!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("m", [8, 11])
def test_gloo_two_rank_four_step_1d(m):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_1d, args=(r, 2, port, m, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=60) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0] <= 1e-13 and res[1] <= 1e-13, res


def test_block_layout_roundtrip():
    a = np.arange(4 * 16).reshape(4, 16)
    blocks = _rows_blocked(a, 4)
    assert blocks.shape == (4, 4, 4)
    assert np.array_equal(blocks[2], a[:, 8:12])
    assert np.array_equal(_unblock(blocks), a)
    # the library's flat map: element (row, v) at ((v >> sh) * SN + row) << sh | (v & (SM-1))
    SN, SM, sh = 4, 4, 2
    flat = blocks.ravel()
    for row in range(SN):
        for v in range(16):
            assert flat[(((v >> sh) * SN + row) << sh) | (v & (SM - 1))] == a[row, v]


def _fused_schedule(grids, P, H):
    """The fused schedule of run_dist_2d_fused written out on flat per-rank
    buffers with the library's pointer arithmetic: rank q's receive slab of
    phase ph, block position r at r * SN * SM, element (row, x) of a block at
    (row << sh) | (x & (SM - 1)); the row pass of rank r stores block q there,
    the final pass of rank r loads it back from the same place."""
    N, M = grids[0].shape
    SN, SM = N // P, M // P
    sh = SM.bit_length() - 1
    blk = SN * SM
    recv = np.zeros((2, P, N * SM), dtype=complex)  # [phase][rank] column slabs
    outs = []
    for g, f in enumerate(grids):
        ph = g & 1
        out = np.zeros((N, M), dtype=complex)
        for r in range(P):  # 1. rows, peer stores
            rows = np.stack([oracle.fft(x) * M for x in f[r * SN:(r + 1) * SN]])
            for row in range(SN):
                for x in range(M):
                    recv[ph, x >> sh, r * blk + ((row << sh) | (x & (SM - 1)))] = rows[row, x]
        for q in range(P):  # 2. columns of rank q's slab, filter columns q SM ..
            cs = recv[ph, q].reshape(N, SM)
            cf = np.stack([oracle.fft(cs[:, j]) for j in range(SM)], axis=1) * H[:, q * SM:(q + 1) * SM] / M
            recv[ph, q] = np.stack([oracle.ifft(cf[:, j]) for j in range(SM)], axis=1).ravel()
        for r in range(P):  # 3. rows, peer loads
            for row in range(SN):
                line = np.array([recv[ph, x >> sh, r * blk + ((row << sh) | (x & (SM - 1)))] for x in range(M)])
                out[r * SN + row] = oracle.ifft(line)
        outs.append(out)
    return outs


@pytest.mark.parametrize("P,N,M", [(2, 8, 16), (4, 16, 8), (8, 16, 16)])
def test_fused_peer_schedule_index_maps(P, N, M):
    """CPU pin of the fused all-to-all addressing (three grids: both receive
    phases, then phase 0 again, each must be independent)."""
    grids = [fixtures.complex_input(N * M, fixtures.UNIFORM, seed=40 + i, dtype=np.complex128).reshape(N, M)
             for i in range(3)]
    H = oracle.gauss_filter(N, M, 0.1)
    for f, out in zip(grids, _fused_schedule(grids, P, H)):
        assert oracle.rel_l2(out, oracle.gauss_pipeline(f, 0.1)) <= 1e-13


def _dist_transpose(src, R, Cn, Cb):
    """k_dist_transpose's addressing over P rank slabs (flat arrays): global
    element (gr, gc) read from src[gr >> rsh][(gr & (R-1)) * Cn + gc],
    written to dst[gc >> bsh][(gc & (Cb-1)) * P R + gr]."""
    P = len(src)
    rsh, bsh = R.bit_length() - 1, Cb.bit_length() - 1
    Rg = P * R
    dst = [np.zeros(Cb * Rg, dtype=complex) for _ in range(P)]
    gr = np.arange(Rg)[:, None]
    gc = np.arange(Cn)[None, :]
    vals = np.stack(src)[gr >> rsh, (gr & (R - 1)) * Cn + gc]
    d = np.broadcast_to(gc >> bsh, vals.shape)
    off = (gc & (Cb - 1)) * Rg + gr
    for q in range(P):
        sel = d == q
        dst[q][off[sel]] = vals[sel]
    return dst


@pytest.mark.parametrize("P,m", [(2, 6), (4, 8), (8, 9)])
def test_fused_four_step_index_maps(P, m):
    """CPU pin of the fused distributed four-step (run_dist_1d_fused): three
    cross-rank transposes with the kernel's addressing around the oracle's
    sub-FFTs and the four-step twiddle equal the oracle's 1D transform."""
    n = 1 << m
    N1, N2 = 1 << (m - m // 2), 1 << (m // 2)
    S1, S2 = N1 // P, N2 // P
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=31, dtype=np.complex128)
    slabs = [x[r * n // P:(r + 1) * n // P] for r in range(P)]
    a = _dist_transpose(slabs, S2, N1, S1)  # rank q: [S1][N2], rows n1
    for r in range(P):
        A = a[r].reshape(S1, N2)
        A = np.stack([oracle.fft(row) * N2 for row in A])
        n1 = r * S1 + np.arange(S1)[:, None]
        A = A * np.exp(-2j * np.pi * ((n1 * np.arange(N2)[None, :]) % n) / n)
        a[r] = A.ravel()
    bb = _dist_transpose(a, S1, N2, S2)  # rank q: [S2][N1], rows k2
    for r in range(P):
        B = bb[r].reshape(S2, N1)
        bb[r] = (np.stack([oracle.fft(row) * N1 for row in B]) / n).ravel()
    out = _dist_transpose(bb, S2, N1, S1)  # rank q: X[q n/P, ..)
    assert oracle.rel_l2(np.concatenate(out), oracle.fft(x)) <= 1e-13


# ---------------------------------------------- NEXT-2: the paper's tree
def _branches(x, P):
    """Rank q's branch = the cyclic subsequence x[q + P j]."""
    return np.concatenate([x[q::P] for q in range(P)])


@pytest.mark.gpu
@pytest.mark.parametrize("P", [1, 2, 4, 8])
@pytest.mark.parametrize("m", [3, 10, 16, 20])
def test_virtual_ranks_paper_tree(P, m):
    """fft_forward_paper_tree on P virtual ranks: branch FFTs of the cyclic
    subsequences, log2 P combine rounds, the MASTER's vector = (1/n) DFT."""
    b = _lib()
    n = 1 << m
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=800 + m)
    p = b.Plan((n,), batch=1)
    if P > 1:
        p.set_virtual_ranks(P)
    xd = torch.from_numpy(_branches(x, P)).cuda()
    out = torch.empty(n, dtype=torch.complex64, device="cuda")
    p.forward_paper_tree(xd, out)
    torch.cuda.synchronize()
    p.destroy()
    assert oracle.rel_l2(out.cpu().numpy(), oracle.fft(x)) <= 1e-5


@pytest.mark.gpu
def test_paper_tree_nccl_single_rank():
    """The NCCL branch of the schedule with a 1-rank communicator (no rounds)."""
    b = _lib()
    n = 1 << 14
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=810)
    p = b.Plan((n,), batch=1)
    p.set_comm(b.nccl_unique_id(), 1, 0)
    out = torch.empty(n, dtype=torch.complex64, device="cuda")
    p.forward_paper_tree(torch.from_numpy(x).cuda(), out)
    torch.cuda.synchronize()
    p.destroy()
    assert oracle.rel_l2(out.cpu().numpy(), oracle.fft(x)) <= 1e-5


def _worker_tree(rank, world, port, m, q):
    """The library's tree protocol (plan.cu run_paper_tree) with numpy local
    steps and gloo point-to-point messages: round S sends q + S/2 -> q."""
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        P, n = world, 1 << m
        x = fixtures.complex_input(n, fixtures.NORMAL, seed=33, dtype=np.complex128)
        v = oracle.fft(x[rank::P])  # branch, with its 1/len
        S = P
        while S > 1:
            if rank >= S:
                break
            if rank >= S // 2:
                dist.send(torch.from_numpy(np.ascontiguousarray(v)), rank - S // 2)
                break
            o = torch.empty(v.size, dtype=torch.complex128)
            dist.recv(o, rank + S // 2)
            M = v.size
            w = np.exp(-2j * np.pi * np.arange(M) / (2 * M))
            v = np.concatenate([(v + w * o.numpy()) / 2, (v - w * o.numpy()) / 2])
            S //= 2
        q.put((rank, oracle.rel_l2(v, oracle.fft(x)) if rank == 0 else 0.0))
    except Exception as exc:
        q.put((rank, f"error: {exc!r}"))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gloo_paper_tree_protocol(world):
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_tree, args=(r, world, port, 10, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=90) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    assert res[0] <= 1e-13, res


@pytest.mark.gpu
def test_virtual_rank_count_change_rebuilds_the_four_step():
    """Changing the rank count after a first distributed call rebuilds the
    four-step sub-plans (their batches are N1 / P and N2 / P): P = 2, then 4,
    then 1 (the local path), each against the oracle."""
    b = _lib()
    n = 1 << 16
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=640, dtype=np.complex64)
    ref = oracle.fft(x)
    p = b.Plan((n,), batch=1)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    for P in (2, 4, 1):
        p.set_virtual_ranks(P)
        p.forward(xd, yd)
        torch.cuda.synchronize()
        assert oracle.rel_l2(yd.cpu().numpy(), ref) <= 1e-5, P
    p.destroy()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["2d", "1d"])
def test_phase_timing(kind):
    """fft_plan_set_profiling / fft_plan_phase_times: one labelled device time
    per phase of the distributed schedules (the exchange phases carry
    "exchange"), one phase for a local call, none when profiling is off."""
    b = _lib()
    if kind == "2d":
        N = M = 1024
        p = b.Plan((N, M), batch=1)
        p.set_virtual_ranks(4)
        x = torch.from_numpy(fixtures.complex_input(N * M, 0, seed=650).reshape(N, M)).cuda()
        run = lambda: p.filter_pipeline(x, torch.empty_like(x), b.FILTER_GAUSS, 0.1)  # noqa: E731
    else:
        n = 1 << 20
        p = b.Plan((n,), batch=1)
        p.set_virtual_ranks(4)
        x = torch.from_numpy(fixtures.complex_input(n, 1, seed=651)).cuda()
        run = lambda: p.forward(x, torch.empty_like(x))  # noqa: E731
    run()
    assert p.phase_times() == []
    p.set_profiling(True)
    run()
    ph = p.phase_times()
    assert len(ph) >= 3 and all(t >= 0.0 for _, t in ph)
    assert any("exchange" in lab for lab, _ in ph) and all(lab for lab, _ in ph)
    q = b.Plan((4096,), batch=8)
    q.set_profiling(True)
    y = torch.from_numpy(fixtures.complex_input(8 * 4096, 1, seed=652)).cuda()
    q.forward(y, torch.empty_like(y))
    assert [lab for lab, _ in q.phase_times()] == ["forward"]
    p.destroy()
    q.destroy()
