"""CUDA-graph capture of the library's calls (the launch-bound configs -- C1,
NEXT-1 -- are meant to be replayed from graphs; B200 design rule: "capture
launch-bound inner loops in CUDA graphs").  Each case warms the plan up once
(first-call allocations and kernel attributes happen outside the capture),
captures the call(s) on the plan's stream, then replays the graph on fresh
inputs copied into the captured input buffer and compares with the oracle.
Replayed more than once, so state a launch would carry on the host (a
counter target, a receive phase) would show up as wrong results: the
cooperative two-pass pipeline's grid barrier (k_rows_tma2) resets itself,
the task pipelines' counters are reset by captured memsets."""
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

    return lib


def _capture(stream, fn):
    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("n,batch,prec", [(1024, 1, "c128"), (4096, 64, "c64"), (65536, 40, "c64"),
                                          (1 << 20, 1, "c64")])
def test_graph_1d_forward_inverse(b, n, batch, prec):
    """1D forward (1/N) then inverse in one graph: C1's k_rows, the TMA row
    kernel, C2's cooperative task pipeline (k_ab_st: counters memset and the
    L2 access-policy window inside the capture), the multi-pass Stockham."""
    dt = np.complex128 if prec == "c128" else np.complex64
    st = torch.cuda.Stream()
    p = b.Plan((n,), batch=batch, precision=b.C128 if prec == "c128" else b.C64, stream=st)
    xd = torch.empty((batch, n), dtype=torch.complex128 if prec == "c128" else torch.complex64, device="cuda")
    yd, zd = torch.empty_like(xd), torch.empty_like(xd)

    def step():
        p.forward(xd, yd)
        p.inverse(yd, zd)

    step()
    g = _capture(st, step)
    tol = 1e-12 if prec == "c128" else 1e-5
    for seed in (11, 12, 13):
        x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=seed + n % 97, dtype=dt).reshape(batch, n)
        xd.copy_(torch.from_numpy(x))
        g.replay()
        torch.cuda.synchronize()
        assert oracle.rel_l2(yd.cpu().numpy(), oracle.fft_batch(x)) <= tol
        assert oracle.rel_l2(zd.cpu().numpy(), x) <= tol
    p.destroy()


@pytest.mark.parametrize("real_out", [False, True])
def test_graph_c3_pipeline(b, real_out):
    """C3's Gaussian pipeline on a 2048^2 real image: complex output = the
    one cooperative launch with the self-resetting grid barrier; real output
    = two launches, the second a programmatic dependent launch."""
    N = 2048
    st = torch.cuda.Stream()
    p = b.Plan((N, N), batch=1, precision=b.C64,
               flags=b.IN_REAL_F32 | (b.OUT_REAL_F32 if real_out else 0), stream=st)
    idev = torch.empty((N, N), dtype=torch.float32, device="cuda")
    out = torch.empty((N, N), dtype=torch.float32 if real_out else torch.complex64, device="cuda")

    def step():
        p.filter_pipeline(idev, out, b.FILTER_GAUSS, 0.1)

    step()
    g = _capture(st, step)
    for seed in (21, 22, 23):
        img = fixtures.sky_image(N, N, seed=seed)
        idev.copy_(torch.from_numpy(img))
        g.replay()
        torch.cuda.synchronize()
        ref = oracle.gauss_pipeline(img.astype(np.complex128), 0.1)
        got = out.cpu().numpy()
        assert oracle.rel_l2(got, ref.real if real_out else ref) <= 1e-5
    p.destroy()


def test_graph_long_column_pipeline(b):
    """8192-row grids: the row filter pass then the one-pass column filter
    k_colfilt (task pipeline, counters memset inside the capture)."""
    N, M = 8192, 256
    st = torch.cuda.Stream()
    p = b.Plan((N, M), batch=1, stream=st)
    fd = torch.empty((N, M), dtype=torch.complex64, device="cuda")
    od = torch.empty_like(fd)
    p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    g = _capture(st, lambda: p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1))
    for seed in (31, 32):
        f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=seed).reshape(N, M)
        fd.copy_(torch.from_numpy(f))
        g.replay()
        torch.cuda.synchronize()
        assert oracle.rel_l2(od.cpu().numpy(), oracle.gauss_pipeline(f, 0.1)) <= 1e-5
    p.destroy()


def test_graph_image_application(b):
    """NEXT-1 (the paper's Sec. 6 application) replayed from a graph: the
    same bytes as the direct call."""
    st = torch.cuda.Stream()
    p = b.Plan((512, 512), batch=1, precision=b.C64, stream=st)
    idev = torch.empty((506, 460), dtype=torch.uint8, device="cuda")
    out = torch.empty_like(idev)
    spec = torch.empty((512, 512), dtype=torch.float32, device="cuda")

    def step():
        p.image_filter_u8(idev, out, b.FILTER_IDEAL_LITERAL, 340.0, 255, spec)

    step()
    g = _capture(st, step)
    for seed in (41, 42):
        img = fixtures.sky_image_u8(506, 460, seed=seed)
        idev.copy_(torch.from_numpy(img))
        step()
        torch.cuda.synchronize()
        ref, sref = out.clone(), spec.clone()
        out.zero_()
        spec.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert torch.equal(spec, sref)
    p.destroy()
