"""GPU parity of the end-to-end host-buffer entry point fft_execute_host
(include/b200fft.h): host -> device copies, the transform, device -> host,
pipelined over batch chunks on two streams that share the plan's workspace
(the C2 ring and counters, the 2D intermediate grid, the pass ping-pong
buffer).  Every case spans several 64 MiB chunks with a ragged last one, and
is compared with the oracle over the whole output."""
import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0103001_b200 as lib

    lib.load_library()
    return lib


def pinned(a):
    t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    return t


@pytest.mark.parametrize("n,batch", [(65536, 520), (1 << 20, 70), (4096, 20000)])
def test_execute_host_1d(b, n, batch):
    """C2's kernel (128 rows per chunk: 5 chunks, the last of 8 rows), the
    multi-pass path (8 rows per chunk) and the single-CTA path, forward and
    inverse, pinned and pageable host buffers."""
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=1200 + batch).reshape(batch, n)
    p = b.Plan((n,), batch=batch)
    hin = pinned(x)
    hout = torch.empty_like(hin).pin_memory()
    p.execute_host(+1, hin, hout)
    y = hout.numpy().copy()
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= 1e-5
    back = np.empty_like(x)  # pageable output
    p.execute_host(-1, y, back)
    assert oracle.rel_l2(back, oracle.fft_batch(y, inverse=True)) <= 1e-5
    assert oracle.rel_l2(back, x) <= 1e-5
    p.destroy()


def test_execute_host_after_device_work(b):
    """execute_host is ordered after work already queued on the plan's
    stream, and repeated calls reuse the staging buffers."""
    n, batch = 65536, 300
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=1250).reshape(batch, n)
    p = b.Plan((n,), batch=batch, stream=torch.cuda.current_stream())
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    hin, hout = pinned(x), torch.empty(batch, n, dtype=torch.complex64).pin_memory()
    for _ in range(2):
        p.execute_host(+1, hin, hout)
    torch.cuda.synchronize()
    assert oracle.rel_l2(hout.numpy(), yd.cpu().numpy()) <= 1e-6
    p.destroy()


@pytest.mark.parametrize("real", [False, True])
def test_execute_host_batched_pipeline(b, real):
    """Batched 2D Gaussian pipeline (512^2 grids, 32 per chunk: 2 chunks, the
    second ragged) on host buffers, complex or float32 input, against the
    oracle grid by grid."""
    N = M = 512
    batch = 40
    if real:
        f = np.stack([fixtures.sky_image(N, M, seed=1300 + i, nsrc=30) for i in range(batch)])
        flags = b.IN_REAL_F32
    else:
        f = fixtures.complex_input(batch * N * M, fixtures.UNIFORM, seed=1300).reshape(batch, N, M)
        flags = 0
    p = b.Plan((N, M), batch=batch, flags=flags)
    hin = pinned(f)
    hout = torch.empty(batch, N, M, dtype=torch.complex64).pin_memory()
    p.execute_host(0, hin, hout, b.FILTER_GAUSS, 0.1)
    out = hout.numpy()
    ref = np.stack([oracle.gauss_pipeline(f[i].astype(np.complex128), 0.1) for i in range(batch)])
    assert oracle.rel_l2(out, ref) <= 1e-5
    p.destroy()


def test_execute_host_batched_2d_forward_inverse(b):
    N, M, batch = 256, 1024, 70
    f = fixtures.complex_input(batch * N * M, fixtures.UNIFORM, seed=1350).reshape(batch, N, M)
    p = b.Plan((N, M), batch=batch)
    F = np.empty_like(f)
    p.execute_host(+1, f, F)
    ref = np.stack([oracle.fft2d(f[i]) for i in range(batch)])
    assert oracle.rel_l2(F, ref) <= 1e-5
    g = np.empty_like(f)
    p.execute_host(-1, F, g)
    assert oracle.rel_l2(g, f) <= 1e-5
    p.destroy()
