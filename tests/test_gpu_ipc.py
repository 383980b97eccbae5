"""The cross-process data plane of the fused multi-rank schedules (H9,
PAPER.md P:196-224: the paper's processor-to-processor sends, here one
process per rank writing into the other ranks' receive slabs), run by
several PROCESSES on one GPU.

NCCL refuses two ranks on one device, so the plans take the two collectives
of the fused schedules -- the CUDA-IPC handle all-gather and the barriers --
from host callbacks over a gloo process group
(``fft_plan_set_host_collectives``); each barrier first drains the plan's
stream, so no kernel ever waits on another process (B200_PROFILING.md: ranks
on one GPU must not spin on each other).  Everything else is the
``fft_plan_set_comm`` path: receive slabs allocated per rank and mapped into
every other process with ``cudaIpcOpenMemHandle``, the row / transpose
kernels storing into (and the last pass loading from) the other processes'
slabs, the slab layouts, column offsets and scales.  Each rank's local slab
is compared with the oracle's full-size result."""
import multiprocessing as mp
import os
import socket
import traceback

import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_cs_0103001_b200 as b

        torch.cuda.set_device(0)

        def allgather(mine):
            out = [None] * world
            dist.all_gather_object(out, mine)
            return out

        res = {}
        if case[0] == "2d":
            _, N, M, batch = case
            SN = N // world
            f = fixtures.complex_input(batch * N * M, fixtures.UNIFORM, seed=31 + N + M).reshape(batch, N, M)
            p = b.Plan((N, M), batch=batch)
            p.set_host_collectives(world, rank, allgather, dist.barrier)
            fd = torch.from_numpy(np.ascontiguousarray(f[:, rank * SN:(rank + 1) * SN])).cuda()
            od = torch.empty_like(fd)
            for _ in range(3):  # both receive phases and back
                p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
            torch.cuda.synchronize()
            res["pipe"] = od.cpu().numpy()
            F, G = torch.empty_like(fd), torch.empty_like(fd)
            p.forward(fd, F)
            p.inverse(fd, G)
            torch.cuda.synchronize()
            res["fwd"], res["inv"] = F.cpu().numpy(), G.cpu().numpy()
            res["launches"] = p.last_launch_count()
        elif case[0] == "c5":
            # BASELINE configs[4]: 2^30 over the processes (32768 x 32768
            # four-step, 32768-point sub-FFTs with the fused outer twiddle);
            # each rank returns the sampled bins it owns
            _, bins_f, bins_i = case
            n = 1 << 30
            loc = n // world
            x = np.empty(loc, np.complex64)
            p = b.Plan((n,), batch=1)
            p.set_host_collectives(world, rank, allgather, dist.barrier)
            for name, seed, bins, fwd in (("fwd", 5, bins_f, True), ("inv", 105, bins_i, False)):
                fixtures.complex_input(loc, fixtures.NORMAL, seed=seed, offset=rank * loc, out=x)
                xd = torch.from_numpy(x).cuda()
                yd = torch.empty_like(xd)
                (p.forward if fwd else p.inverse)(xd, yd)
                torch.cuda.synchronize()
                mine = [int(k) for k in bins if rank * loc <= k < (rank + 1) * loc]
                idx = torch.tensor([k - rank * loc for k in mine], dtype=torch.int64, device="cuda")
                res[name] = dict(zip(mine, yd[idx].cpu().numpy().tolist()))
                del xd, yd
        else:
            _, m = case
            n = 1 << m
            loc = n // world
            x = fixtures.complex_input(n, fixtures.NORMAL, seed=40 + m)
            p = b.Plan((n,), batch=1)
            p.set_host_collectives(world, rank, allgather, dist.barrier)
            xd = torch.from_numpy(x[rank * loc:(rank + 1) * loc].copy()).cuda()
            yd, zd = torch.empty_like(xd), torch.empty_like(xd)
            for _ in range(2):  # both receive phases
                p.forward(xd, yd)
                p.inverse(xd, zd)
            torch.cuda.synchronize()
            res["fwd"], res["inv"] = yd.cpu().numpy(), zd.cpu().numpy()
        p.destroy()
        q.put((rank, res))
    except Exception:  # report instead of hanging the parent
        q.put((rank, "error: " + traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def _run(world, case):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    try:
        res = dict(q.get(timeout=600) for _ in procs)
    finally:
        for pr in procs:
            pr.join(timeout=120)
            if pr.exitcode is None:
                pr.kill()
    for r in range(world):
        assert not isinstance(res[r], str), res[r]
    return res


@pytest.mark.parametrize("world,N,M,batch", [(2, 1024, 1024, 1), (4, 512, 256, 2), (2, 8192, 256, 1)])
def test_processes_fused_2d_schedule(world, N, M, batch):
    """Row slabs -> peer stores into the other processes' column slabs ->
    columns (for N = 8192 the one-pass k_colfilt with the slab's column
    offset into g_M) -> peer loads back; the Gaussian pipeline, the forward
    and the inverse 2D DFT (eq5 / 2D-IDFT), three calls so both
    receive phases are used."""
    res = _run(world, ("2d", N, M, batch))
    f = fixtures.complex_input(batch * N * M, fixtures.UNIFORM, seed=31 + N + M).reshape(batch, N, M)
    got = {k: np.concatenate([res[r][k] for r in range(world)], axis=1) for k in ("pipe", "fwd", "inv")}
    for i in range(batch):
        assert oracle.rel_l2(got["pipe"][i], oracle.gauss_pipeline(f[i], 0.1)) <= 1e-5
        assert oracle.rel_l2(got["fwd"][i], oracle.fft2d(f[i])) <= 1e-5
        assert oracle.rel_l2(got["inv"][i], oracle.ifft2d(f[i])) <= 1e-5


@pytest.mark.parametrize("world,m", [(2, 20), (4, 16)])
def test_processes_fused_four_step_1d(world, m):
    """One transform of n = 2^m over the processes (C5's schedule): three
    cross-process transposes (stores into the peers' receive slabs, the last
    a pull from them) around the sub-FFT batches, three barriers; natural
    order, forward (1/n) and inverse."""
    res = _run(world, ("1d", m))
    x = fixtures.complex_input(1 << m, fixtures.NORMAL, seed=40 + m)
    fwd = np.concatenate([res[r]["fwd"] for r in range(world)])
    inv = np.concatenate([res[r]["inv"] for r in range(world)])
    assert oracle.rel_l2(fwd, oracle.fft(x)) <= 1e-5
    assert oracle.rel_l2(inv, oracle.ifft(x)) <= 1e-5


def test_processes_c5_shape():
    """C5's shape (n = 2^30) over 2 processes: forward on seed 5 and inverse
    on seed 105, 64 bins each against the oracle's direct sums (SURVEY 8(c)
    O7) -- the distributed four-step with the 32768-point one-pass sub-FFTs
    and the cross-process transposes."""
    n = 1 << 30
    rng_f, rng_i = np.random.default_rng(5), np.random.default_rng(105)
    bins_f = np.concatenate([[0, 1, n // 2, n - 1], rng_f.integers(0, n, 60)]).astype(np.int64)
    bins_i = np.concatenate([[0, 1, n // 2, n - 1], rng_i.integers(0, n, 60)]).astype(np.int64)
    res = _run(2, ("c5", bins_f.tolist(), bins_i.tolist()))
    x = np.empty(n, np.complex64)
    for name, seed, bins, inv in (("fwd", 5, bins_f, False), ("inv", 105, bins_i, True)):
        got = {}
        for r in range(2):
            got.update(res[r][name])
        fixtures.complex_input(n, fixtures.NORMAL, seed=seed, out=x)
        ref = oracle.dft_bins(x, bins, inverse=inv)
        assert oracle.rel_l2(np.array([got[int(k)] for k in bins]), ref) <= 1e-5
