"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle,
element by element on the same seeded inputs.

Tolerances (BASELINE.json north_star): relative L2 over the whole output
<= 1e-5 for complex64 and <= 1e-12 for complex128.
"""
import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.complex64: 1e-5, np.complex128: 1e-12}


@pytest.fixture(scope="module")
def fft():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0103001_b200 as b

    b.load_library()
    return b


def prec_of(dtype):
    import paper_cs_0103001_b200 as b

    return b.C64 if dtype == np.complex64 else b.C128


def run_1d(b, x, inverse=False):
    batch, n = x.shape
    p = b.Plan((n,), batch=batch, precision=prec_of(x.dtype.type))
    p.set_stream(torch.cuda.current_stream())
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    (p.inverse if inverse else p.forward)(xd, yd)
    torch.cuda.synchronize()
    out = yd.cpu().numpy()
    p.destroy()
    return out


# ------------------------------------------------------------------- 1D
@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("m", range(0, 14))
@pytest.mark.parametrize("batch", [1, 3, 64])
def test_1d_single_pass_sizes(fft, dtype, m, batch):
    n = 1 << m
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=100 + m, dtype=dtype).reshape(batch, n)
    y = run_1d(fft, x)
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= TOL[dtype]
    z = run_1d(fft, x, inverse=True)
    assert oracle.rel_l2(z, oracle.fft_batch(x, inverse=True)) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("m", [14, 15, 16, 17, 18, 20, 21, 22])
def test_1d_multi_pass_sizes(fft, dtype, m):
    n = 1 << m
    batch = 2 if m <= 20 else 1
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=200 + m, dtype=dtype).reshape(batch, n)
    y = run_1d(fft, x)
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= TOL[dtype]
    z = run_1d(fft, x, inverse=True)
    assert oracle.rel_l2(z, oracle.fft_batch(x, inverse=True)) <= TOL[dtype]


def test_1d_three_pass_radix512(fft):
    """2^27 = 512^3: three pipelined passes (k_pass_pipe), the last one with a
    two-level pass twiddle (pa x pb), forward and inverse against the oracle."""
    n = 1 << 27
    x = fixtures.complex_input(n, fixtures.NORMAL, seed=227).reshape(1, n)
    assert oracle.rel_l2(run_1d(fft, x), oracle.fft_batch(x)) <= TOL[np.complex64]
    assert oracle.rel_l2(run_1d(fft, x, inverse=True), oracle.fft_batch(x, inverse=True)) <= TOL[np.complex64]


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
def test_1d_65536_multipass_fallback(fft, dtype, monkeypatch):
    """The generic 2-pass schedule for N = 65536 (the one-pass cluster kernel
    is disabled at plan creation) against the oracle."""
    monkeypatch.setenv("B200FFT_NO_CLUSTER", "1")
    x = fixtures.complex_input(3 * 65536, fixtures.NORMAL, seed=216, dtype=dtype).reshape(3, 65536)
    assert oracle.rel_l2(run_1d(fft, x), oracle.fft_batch(x)) <= TOL[dtype]
    assert oracle.rel_l2(run_1d(fft, x, inverse=True), oracle.fft_batch(x, inverse=True)) <= TOL[dtype]


@pytest.mark.parametrize("case", ["1d-8", "1d-2048", "1d-8192", "1d-32768", "1d-65536", "1d-65536pair",
                                  "1d-2^17", "1d-2^21",
                                  "2d-256x512", "pipe-2048-real", "pipe-8192x16", "pipe-literal",
                                  "dist2d-4", "dist1d-4"])
def test_no_writes_outside_the_buffers(fft, case, monkeypatch):
    """Canary bounds check (compute-sanitizer is not available on this pool):
    every call runs on the interior of a buffer whose 64 KiB guard zones on
    both sides hold a sentinel, for output and input; the guards must come
    back untouched and the input unchanged when out != in."""
    import paper_cs_0103001_b200 as b

    G = 8192  # guard elements (complex64) = 64 KiB
    kind, _, rest = case.partition("-")

    def guarded(n, dtype=torch.complex64):
        buf = torch.full((n + 2 * G,), complex(1.2345e6, -6.789e5), dtype=dtype, device="cuda")
        return buf, buf[G:G + n]

    def check(buf, n):
        ref = torch.tensor(complex(1.2345e6, -6.789e5), dtype=buf.dtype)
        assert bool((buf[:G].cpu() == ref).all()) and bool((buf[G + n:].cpu() == ref).all())

    if kind == "1d":
        if rest == "65536pair":  # k_ab_pair (C2 with Y in TMEM)
            monkeypatch.setenv("B200FFT_C2", "pair")
            rest = "65536"
        n = {"8": 8, "2048": 2048, "8192": 8192, "32768": 32768, "65536": 65536, "2^17": 1 << 17,
             "2^21": 1 << 21}[rest]
        batch = 3 if n <= 65536 else (2 if n < (1 << 21) else 1)
        p = b.Plan((n,), batch=batch)
        shapes = [(n * batch, lambda x, y: p.forward(x, y)), (n * batch, lambda x, y: p.inverse(x, y))]
    elif kind == "dist1d":
        n = 1 << 16
        p = b.Plan((n,), batch=1)
        p.set_virtual_ranks(4)
        shapes = [(n, lambda x, y: p.forward(x, y))]
    elif kind == "2d" or kind == "dist2d":
        N, M = (256, 512)
        p = b.Plan((N, M))
        if kind == "dist2d":
            p.set_virtual_ranks(4)
        shapes = [(N * M, lambda x, y: p.forward(x, y)),
                  (N * M, lambda x, y: p.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1))]
    else:  # pipelines
        if rest == "2048-real":
            N = M = 2048
            p = b.Plan((N, M), flags=b.IN_REAL_F32)
            fin = torch.full((N * M + 2 * G,), 7.5, device="cuda")
            fin[G:G + N * M] = torch.rand(N * M, device="cuda")
            obuf, o = guarded(N * M)
            before = fin.clone()
            p.filter_pipeline(fin[G:G + N * M], o, b.FILTER_GAUSS, 0.1)
            torch.cuda.synchronize()
            check(obuf, N * M)
            assert torch.equal(fin, before)
            return
        if rest == "8192x16":
            N, M = 8192, 16
            p = b.Plan((N, M))
        else:
            N, M = 128, 64
            p = b.Plan((N, M))
        shapes = [(N * M, lambda x, y: p.filter_pipeline(x, y, b.FILTER_IDEAL_LITERAL if rest == "literal"
                                                         else b.FILTER_GAUSS, 30.0 if rest == "literal" else 0.1))]
    for n, call in shapes:
        ibuf, x = guarded(n)
        x.copy_(torch.randn(n, dtype=torch.complex64, device="cuda"))
        obuf, y = guarded(n)
        before = ibuf.clone()
        call(x, y)
        torch.cuda.synchronize()
        check(obuf, n)
        assert torch.equal(ibuf, before)  # out != in: the input is read only
    p.destroy()


def test_c1_config(fft):
    """BASELINE configs[0]: N=1024, batch 1, complex128, U[-1,1], seed 1;
    forward (1/N) then inverse round trip."""
    x = fixtures.complex_input(1024, fixtures.UNIFORM, seed=1, dtype=np.complex128).reshape(1, 1024)
    y = run_1d(fft, x)
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= 1e-12
    z = run_1d(fft, y, inverse=True)
    assert oracle.rel_l2(z, x) <= 1e-12


def test_impulse_is_exact(fft):
    # delta_0 -> flat 1/N exactly (F2: the power-of-two scale is exact)
    for n in (16, 1024, 8192, 65536):
        x = np.zeros((1, n), np.complex64)
        x[0, 0] = 1
        y = run_1d(fft, x)
        assert np.array_equal(y, np.full((1, n), 1.0 / n, np.complex64))


def test_inplace_and_empty(fft):
    import paper_cs_0103001_b200 as b

    for n in (256, 65536, 1 << 21):
        x = fixtures.complex_input(n, fixtures.NORMAL, seed=7).reshape(1, n)
        p = b.Plan((n,), batch=1)
        xd = torch.from_numpy(x).cuda()
        p.forward(xd)  # out == in
        torch.cuda.synchronize()
        assert oracle.rel_l2(xd.cpu().numpy(), oracle.fft_batch(x)) <= 1e-5
    p0 = b.Plan((256,), batch=0)
    p0.forward(torch.empty(1, dtype=torch.complex64, device="cuda"))
    torch.cuda.synchronize()


def test_c2_full_size_whole_output(fft):
    """BASELINE configs[1]: 4096 x 65536 complex64, N(0,1), seed 2, in the
    launch configuration bench.py times.  The forward output is compared with
    the oracle over ALL 4096 rows (one whole-output rel-L2, O8); the inverse
    runs on the independent seed-102 input and is compared with
    the oracle's Sec. 3 inverse over all rows; plus the forward -> inverse
    round trip over the whole batch."""
    import paper_cs_0103001_b200 as b

    n, batch = 65536, 4096
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=2).reshape(batch, n)
    p = b.Plan((n,), batch=batch)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    zd = torch.empty_like(xd)
    p.inverse(yd, zd)
    torch.cuda.synchronize()
    err = torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd)
    assert float(err) <= 1e-5
    del zd
    y = yd.cpu().numpy()
    ref = oracle.fft_batch(x)
    e_fwd = oracle.rel_l2(y, ref)
    del ref, y
    assert e_fwd <= 1e-5, e_fwd
    c = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=102).reshape(batch, n)
    xd.copy_(torch.from_numpy(c))
    p.inverse(xd, yd)
    torch.cuda.synchronize()
    f = yd.cpu().numpy()
    ref = oracle.fft_batch(c, inverse=True)
    e_inv = oracle.rel_l2(f, ref)
    assert e_inv <= 1e-5, e_inv
    p.destroy()


# ------------------------------------------------------------------- 2D
def run_2d(b, f, inverse=False):
    N, M = f.shape
    p = b.Plan((N, M), batch=1, precision=prec_of(f.dtype.type))
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    (p.inverse if inverse else p.forward)(fd, od)
    torch.cuda.synchronize()
    p.destroy()
    return od.cpu().numpy()


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("N,M", [(1, 1), (2, 8), (8, 2), (16, 16), (64, 32), (32, 1024), (256, 512),
                                 (4096, 16), (16, 4096), (1024, 1024)])
def test_2d_forward_inverse(fft, dtype, N, M):
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=300 + N + M, dtype=dtype).reshape(N, M)
    F = run_2d(fft, f)
    assert oracle.rel_l2(F, oracle.fft2d(f)) <= TOL[dtype]
    g = run_2d(fft, f, inverse=True)
    assert oracle.rel_l2(g, oracle.ifft2d(f)) <= TOL[dtype]


def test_2d_8192_columns(fft):
    f = fixtures.complex_input(8192 * 16, fixtures.UNIFORM, seed=5).reshape(8192, 16)
    assert oracle.rel_l2(run_2d(fft, f), oracle.fft2d(f)) <= 1e-5


def run_pipeline(b, f, filt, param, real=False):
    N, M = f.shape
    flags = b.IN_REAL_F32 if real else 0
    prec = b.C64 if (real or f.dtype == np.complex64) else b.C128
    p = b.Plan((N, M), batch=1, precision=prec, flags=flags)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty((N, M), dtype=torch.complex64 if prec == b.C64 else torch.complex128, device="cuda")
    p.filter_pipeline(fd, od, filt, param)
    torch.cuda.synchronize()
    p.destroy()
    return od.cpu().numpy()


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("N,M", [(16, 16), (64, 64), (128, 32), (512, 512)])
def test_gauss_pipeline(fft, dtype, N, M):
    import paper_cs_0103001_b200 as b

    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=400 + N, dtype=dtype).reshape(N, M)
    out = run_pipeline(b, f, b.FILTER_GAUSS, 0.1)
    assert oracle.rel_l2(out, oracle.gauss_pipeline(f, 0.1)) <= TOL[dtype]


@pytest.mark.parametrize("N,M", [(64, 64), (128, 32), (2048, 2048)])
def test_gauss_pipeline_literal_three_pass_order(fft, N, M, monkeypatch):
    """The literal order 2D-FFT -> x H -> 2D-IFFT (rows, fused columns, rows),
    i.e. the separable fast path disabled, against the oracle."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_PIPE_LITERAL", "1")
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=410 + N, dtype=np.complex64).reshape(N, M)
    out = run_pipeline(b, f, b.FILTER_GAUSS, 0.1)
    assert oracle.rel_l2(out, oracle.gauss_pipeline(f, 0.1)) <= 1e-5
    img = fixtures.sky_image(256, 256, seed=3, nsrc=20)
    out = run_pipeline(b, img, b.FILTER_GAUSS, 0.1, real=True)
    assert oracle.rel_l2(out, oracle.gauss_pipeline(img.astype(np.complex128), 0.1)) <= 1e-5


def ideal_mask(N, M, b_, literal):
    u = np.arange(N)[:, None]
    v = np.arange(M)[None, :]
    if literal:  # Eq. (filtro): 0 inside radius b of the centre, 1 outside
        return np.where((u - N // 2) ** 2 + (v - M // 2) ** 2 <= b_ * b_, 0.0, 1.0)
    ku = np.where(u < N // 2, u, u - N)
    kv = np.where(v < M // 2, v, v - M)
    return np.where(ku ** 2 + kv ** 2 <= b_ * b_, 1.0, 0.0)


@pytest.mark.parametrize("literal", [True, False])
def test_ideal_filter_pipeline(fft, literal):
    import paper_cs_0103001_b200 as b

    N = M = 512
    f = fixtures.sky_image(N, M, seed=9, nsrc=30)
    radius = 340.0 if literal else 40.0
    kind = b.FILTER_IDEAL_LITERAL if literal else b.FILTER_IDEAL_LOWPASS
    out = run_pipeline(b, f, kind, radius, real=True)
    ref = oracle.filter_pipeline(f.astype(np.complex128), ideal_mask(N, M, radius, literal))
    assert oracle.rel_l2(out, ref) <= 1e-5


def test_c3_config(fft):
    """BASELINE configs[2]: 2048^2 float32 sky image -> 2D FFT -> Gaussian
    (0.1 Nyquist) -> inverse 2D FFT, complex64, against the oracle."""
    import paper_cs_0103001_b200 as b

    img = fixtures.sky_image(2048, 2048, seed=3)
    out = run_pipeline(b, img, b.FILTER_GAUSS, 0.1, real=True)
    ref = oracle.gauss_pipeline(img.astype(np.complex128), 0.1)
    assert oracle.rel_l2(out, ref) <= 1e-5


@pytest.mark.parametrize("realpair", ["1", "0"])
@pytest.mark.parametrize("N,M,batch", [(2048, 2048, 1), (512, 1024, 3), (256, 2048, 2)])
def test_real_input_complex_output_gauss(fft, N, M, batch, realpair, monkeypatch):
    """Real input, complex output, Gaussian: by default two real rows per
    complex line in both passes and an exactly zero imaginary part (DESIGN.md
    R20; the oracle's imaginary part is rounding noise); with
    B200FFT_PIPE_REALPAIR=0 the promoted complex passes.  Both against the
    oracle's complex fp64 pipeline."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_PIPE_REALPAIR", realpair)
    imgs = np.stack([fixtures.sky_image(N, M, seed=810 + i, nsrc=80) for i in range(batch)])
    p = b.Plan((N, M), batch=batch, flags=b.IN_REAL_F32)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty((batch, N, M), dtype=torch.complex64, device="cuda")
    p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    fused = realpair == "1" and N == M and N >= 512  # both passes in one launch (k_rows_tma2)
    assert p.last_launch_count() == (batch if fused else 2 * batch)
    p.destroy()
    out = o.cpu().numpy()
    ref = np.stack([oracle.gauss_pipeline(imgs[i].astype(np.complex128), 0.1) for i in range(batch)])
    assert oracle.rel_l2(out, ref) <= 1e-5
    assert np.abs(ref.imag).max() <= 1e-9 * np.abs(ref.real).max()
    if realpair == "1":
        assert np.all(out.imag == 0)


def test_c4_config_single_gpu(fft):
    """BASELINE configs[3] at P=1: 8192^2 complex64 U[-1,1], seed 4, same
    Gaussian; compared with the oracle over the whole grid."""
    import paper_cs_0103001_b200 as b

    N = 8192
    f = fixtures.complex_input(N * N, fixtures.UNIFORM, seed=4).reshape(N, N)
    out = run_pipeline(b, f, b.FILTER_GAUSS, 0.1)
    ref = oracle.gauss_pipeline(f, 0.1)
    assert oracle.rel_l2(out, ref) <= 1e-5


def c5_bins(n, seed):
    """64 output bins of a 2^30 transform: both ends, the
    middle, and 60 seeded random bins."""
    return np.concatenate([[0, 1, n // 2, n - 1], np.random.default_rng(seed).integers(0, n, 60)]).astype(np.int64)


def test_c5_config_single_gpu_sampled(fft):
    """BASELINE configs[4] at P=1: N = 2^30 complex64, N(0,1).  Forward on
    seed 5 and inverse on the independent seed-105 input, each compared with
    the oracle's direct compensated sums on 64 bins (O7); Parseval and the
    round trip over the whole transform."""
    import paper_cs_0103001_b200 as b

    n = 1 << 30
    x = np.empty(n, np.complex64)
    fixtures.complex_input(n, fixtures.NORMAL, seed=5, out=x)
    p = b.Plan((n,), batch=1)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    torch.cuda.synchronize()
    bins = c5_bins(n, 5)
    got = yd[torch.from_numpy(bins).cuda()].cpu().numpy()
    ref = oracle.dft_bins(x, bins)
    assert oracle.rel_l2(got, ref) <= 1e-5
    # Parseval with the 1/N convention: sum|x|^2 = N sum|X|^2
    sx = float(torch.sum(xd.abs().double() ** 2))
    sX = float(torch.sum(yd.abs().double() ** 2)) * n
    assert abs(sx - sX) / sx < 1e-5
    zd = torch.empty_like(xd)
    p.inverse(yd, zd)
    torch.cuda.synchronize()
    err = torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd)
    assert float(err) <= 1e-5
    del zd
    # inverse on the independent seed-105 input, 64 bins of the Sec. 3 inverse
    fixtures.complex_input(n, fixtures.NORMAL, seed=105, out=x)
    xd.copy_(torch.from_numpy(x))
    p.inverse(xd, yd)
    torch.cuda.synchronize()
    bins = c5_bins(n, 105)
    got = yd[torch.from_numpy(bins).cuda()].cpu().numpy()
    ref = oracle.dft_bins(x, bins, inverse=True)
    assert oracle.rel_l2(got, ref) <= 1e-5
    p.destroy()


@pytest.mark.parametrize("batch", [1, 2, 5, 20, 27, 28, 37, 300])
@pytest.mark.parametrize("kernel", ["ws", "st", "pair"])
def test_c2_kernel_batches_and_inplace(fft, batch, kernel, monkeypatch):
    """The 65536-point one-HBM-pass task pipelines (fft_c2.cuh: k_ab_ws and
    k_ab_st in both stage configurations) at batch
    sizes that leave the persistent grid partly idle or the task order
    without its steady A/B phase (batch < D), forward and inverse,
    out-of-place and in place, against the oracle.  27 / 28 put a B task
    exactly one grid after an A task it depends on (the self-wait that the
    small-batch grid cap of kernels_c2.cu ab_launch_grid removes: without it
    the kernel hangs there)."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_C2", kernel)
    n = 65536
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=900 + batch).reshape(batch, n)
    p = b.Plan((n,), batch=batch)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    zd = yd.clone()
    p.inverse(zd, zd)  # in place
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= 1e-5
    assert oracle.rel_l2(zd.cpu().numpy(), oracle.fft_batch(y, inverse=True)) <= 1e-5
    p.destroy()


@pytest.mark.parametrize("batch", [1, 2, 5, 17, 56, 300])
def test_ab_32768_batches_and_inplace(fft, batch):
    """32768-point rows through the same one-pass task pipeline (k_ab_st<L =
    32768>: n = n1 + 128 n2, 8 A tasks of 16 columns, 8 B tasks of 32 Y rows
    with 128-point DFTs), forward and in-place inverse against the oracle --
    also the sub-FFT length of the distributed 2^30 four-step."""
    import paper_cs_0103001_b200 as b

    n = 32768
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=1900 + batch).reshape(batch, n)
    p = b.Plan((n,), batch=batch)
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    p.forward(xd, yd)
    zd = yd.clone()
    p.inverse(zd, zd)  # in place
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= 1e-5
    assert oracle.rel_l2(zd.cpu().numpy(), oracle.fft_batch(y, inverse=True)) <= 1e-5
    assert p.last_launch_count() == 1
    p.destroy()


def test_c2_two_plans_two_streams(fft):
    """Two plans (each with its own Y-ring workspace) running concurrently on
    two streams, forward on one and inverse on the other."""
    import paper_cs_0103001_b200 as b

    n, batch = 65536, 64
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=950).reshape(batch, n)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    p1, p2 = b.Plan((n,), batch=batch, stream=s1), b.Plan((n,), batch=batch, stream=s2)
    xd = torch.from_numpy(x).cuda()
    torch.cuda.synchronize()
    y1, y2 = torch.empty_like(xd), torch.empty_like(xd)
    for _ in range(3):
        p1.forward(xd, y1)
        p2.inverse(xd, y2)
    torch.cuda.synchronize()
    assert oracle.rel_l2(y1.cpu().numpy(), oracle.fft_batch(x)) <= 1e-5
    assert oracle.rel_l2(y2.cpu().numpy(), oracle.fft_batch(x, inverse=True)) <= 1e-5
    p1.destroy()
    p2.destroy()


@pytest.mark.parametrize("bits", [16, 32, 128, 256, 512, 1024, 4096, 16384])
def test_c2_tuning_variants(fft, bits, monkeypatch):
    """k_ab_st's tuning bits that keep the results (kernels_c2.cu ab_opts:
    static / paired task positions, X store and A load cache policies, the
    recurrence instead of the constant-table step twiddles) against the
    oracle, so every selectable variant of the product kernel is covered."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_ALLOW_WRONG", "1")
    monkeypatch.setenv("B200FFT_AB_XOPTS", str(bits))
    n, batch = 65536, 40
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=960 + bits % 97).reshape(batch, n)
    p = b.Plan((n,), batch=batch)
    xd = torch.from_numpy(x).cuda()
    yd, zd = torch.empty_like(xd), torch.empty_like(xd)
    p.forward(xd, yd)
    p.inverse(yd, zd)
    torch.cuda.synchronize()
    y = yd.cpu().numpy()
    assert oracle.rel_l2(y, oracle.fft_batch(x)) <= 1e-5
    assert oracle.rel_l2(zd.cpu().numpy(), oracle.fft_batch(y, inverse=True)) <= 1e-5
    p.destroy()


@pytest.mark.parametrize("tw", ["0", "1"])
def test_colfilt_twiddle_variants(fft, tw, monkeypatch):
    """k_colfilt with each step-twiddle source (B200FFT_COLFILT_TW: A / A'
    steps from the constant table or by recurrence) on an 8192 x 256
    Gaussian pipeline against the oracle."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_COLFILT_TW", tw)
    N, M = 8192, 256
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=970 + int(tw)).reshape(N, M)
    out = run_pipeline(b, f, b.FILTER_GAUSS, 0.1)
    assert oracle.rel_l2(out, oracle.gauss_pipeline(f, 0.1)) <= 1e-5


@pytest.mark.parametrize("g2", ["1", "0"])
def test_8192_point_rows_both_kernels(fft, g2, monkeypatch):
    """8192-point complex64 rows: the two-group radix-32 k_rows_tma_g (the
    default) and the one-group radix-16 k_rows_tma (B200FFT_ROWS_G2=0), as 2D
    forward / inverse rows on a 64 x 8192 grid and as the row filter pass of
    the 4096 x 8192 Gaussian pipeline, against the oracle."""
    import paper_cs_0103001_b200 as b

    monkeypatch.setenv("B200FFT_ROWS_G2", g2)
    N, M = 64, 8192
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=980).reshape(N, M)
    p = b.Plan((N, M), batch=1)
    fd = torch.from_numpy(f).cuda()
    F, g = torch.empty_like(fd), torch.empty_like(fd)
    p.forward(fd, F)
    p.inverse(F, g)
    torch.cuda.synchronize()
    p.destroy()
    assert oracle.rel_l2(F.cpu().numpy(), oracle.fft2d(f)) <= 1e-5
    assert oracle.rel_l2(g.cpu().numpy(), oracle.ifft2d(F.cpu().numpy())) <= 1e-5
    # the row filter pass (fwd * g * inv) of the long-column Gaussian path
    N = 4096
    f = fixtures.complex_input(N * M, fixtures.UNIFORM, seed=981).reshape(N, M)
    out = run_pipeline(b, f, b.FILTER_GAUSS, 0.1)
    assert oracle.rel_l2(out, oracle.gauss_pipeline(f, 0.1)) <= 1e-5
