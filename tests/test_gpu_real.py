"""GPU parity of the real-data, half-spectrum transforms:
fft_forward_r2c / fft_inverse_c2r (rank 1 and 2, complex64 and complex128)
and the real-to-real filter pipeline through the half spectrum, against the
oracle's rfft2d / irfft2d / rfft_batch / irfft_batch / filter_pipeline_real
(tests/test_oracle_real.py pins those), on seeded inputs."""
import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.complex64: 1e-5, np.complex128: 1e-12}
RDT = {np.complex64: np.float32, np.complex128: np.float64}


@pytest.fixture(scope="module")
def b():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0103001_b200 as lib

    lib.load_library()
    return lib


def prec(b, dt):
    return b.C64 if dt == np.complex64 else b.C128


def real_input(shape, seed, rdt):
    n = int(np.prod(shape))
    z = fixtures.complex_input((n + 1) // 2, fixtures.NORMAL, seed=seed, dtype=np.complex128)
    return np.ascontiguousarray(z.view(np.float64)[:n].reshape(shape).astype(rdt))


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("m", range(1, 14))
@pytest.mark.parametrize("batch", [1, 3, 17])
def test_r2c_c2r_1d(b, dt, m, batch):
    n = 1 << m
    x = real_input((batch, n), 1400 + m, RDT[dt])
    p = b.Plan((n,), batch=batch, precision=prec(b, dt))
    xd = torch.from_numpy(x).cuda()
    hd = torch.empty((batch, n // 2 + 1), dtype=torch.complex64 if dt == np.complex64 else torch.complex128,
                     device="cuda")
    p.forward_r2c(xd, hd)
    back = torch.empty_like(xd)
    p.inverse_c2r(hd, back)
    torch.cuda.synchronize()
    assert oracle.rel_l2(hd.cpu().numpy(), oracle.rfft_batch(x)) <= TOL[dt]
    assert oracle.rel_l2(back.cpu().numpy(), x) <= TOL[dt]  # Sec. 3 inverse of Eq. E2 = identity
    # an independent Hermitian input, with imaginary parts at bins 0 and n/2
    # (a real signal has none: both sides drop them)
    c = fixtures.complex_input(batch * (n // 2 + 1), fixtures.NORMAL, seed=1500 + m,
                               dtype=dt).reshape(batch, n // 2 + 1)
    cd = torch.from_numpy(c).cuda()
    p.inverse_c2r(cd, back)
    torch.cuda.synchronize()
    ref, _ = oracle.irfft_batch(c, n)
    assert oracle.rel_l2(back.cpu().numpy(), ref) <= TOL[dt]
    p.destroy()


SHAPES = [(1, 2), (2, 2), (4, 8), (8, 4), (16, 16), (64, 32), (32, 1024), (256, 512), (2048, 2048),
          (4096, 16), (16, 8192), (8192, 256)]


@pytest.mark.parametrize("dt", [np.complex64, np.complex128])
@pytest.mark.parametrize("N,M", SHAPES)
def test_r2c_c2r_2d(b, dt, N, M):
    if dt == np.complex128 and N > 4096:
        pytest.skip("complex128 columns up to 4096")
    x = real_input((N, M), 1600 + N + M, RDT[dt])
    p = b.Plan((N, M), batch=1, precision=prec(b, dt))
    cdt = torch.complex64 if dt == np.complex64 else torch.complex128
    xd = torch.from_numpy(x).cuda()
    hd = torch.empty((N, M // 2 + 1), dtype=cdt, device="cuda")
    p.forward_r2c(xd, hd)
    back = torch.empty_like(xd)
    p.inverse_c2r(hd, back)
    torch.cuda.synchronize()
    assert oracle.rel_l2(hd.cpu().numpy(), oracle.rfft2d(x)) <= TOL[dt]
    assert oracle.rel_l2(back.cpu().numpy(), x) <= TOL[dt]
    # C2R of an independent consistent half spectrum (the R2C of another image)
    F = oracle.rfft2d(real_input((N, M), 1700 + N + M, np.float64))
    Fd = torch.from_numpy(F.astype(dt)).cuda()
    p.inverse_c2r(Fd, back)
    torch.cuda.synchronize()
    ref, _ = oracle.irfft2d(F.astype(dt).astype(np.complex128), M)
    assert oracle.rel_l2(back.cpu().numpy(), ref) <= TOL[dt]
    assert oracle.rel_l2(Fd.cpu().numpy(), F.astype(dt)) == 0.0  # the 2D inverse leaves `in` unchanged
    p.destroy()


def test_r2c_c2r_2d_batched_8192(b):
    """A batch of two 8192^2 real grids (the C4 size through the half spectrum)."""
    N = M = 8192
    x = np.stack([real_input((N, M), 1800 + i, np.float32) for i in range(2)])
    p = b.Plan((N, M), batch=2)
    xd = torch.from_numpy(x).cuda()
    hd = torch.empty((2, N, M // 2 + 1), dtype=torch.complex64, device="cuda")
    p.forward_r2c(xd, hd)
    back = torch.empty_like(xd)
    p.inverse_c2r(hd, back)
    torch.cuda.synchronize()
    h = hd.cpu().numpy()
    for i in range(2):
        assert oracle.rel_l2(h[i], oracle.rfft2d(x[i])) <= 1e-5
    assert oracle.rel_l2(back.cpu().numpy(), x) <= 1e-5
    p.destroy()


def filt_H(kind, N, M, param):
    if kind == "gauss":
        return oracle.gauss_filter(N, M, param)
    return oracle.ideal_filter(N, M, param, literal=(kind == "literal"))


@pytest.mark.parametrize("kind,param", [("literal", 340.0), ("lowpass", 40.0), ("gauss", 0.1)])
@pytest.mark.parametrize("N,M,batch", [(512, 512, 1), (256, 1024, 2), (1024, 256, 1), (64, 8, 3)])
def test_half_spectrum_pipeline(b, kind, param, N, M, batch, monkeypatch):
    """FFT_IN_REAL_F32 | FFT_OUT_REAL_F32 through the half spectrum, every
    filter (the Gaussian forced onto this path), against the oracle."""
    monkeypatch.setenv("B200FFT_PIPE_HALF", "1")
    kinds = {"literal": b.FILTER_IDEAL_LITERAL, "lowpass": b.FILTER_IDEAL_LOWPASS, "gauss": b.FILTER_GAUSS}
    imgs = np.stack([fixtures.sky_image(N, M, seed=1900 + i, nsrc=30) for i in range(batch)])
    p = b.Plan((N, M), batch=batch, flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty_like(x)
    p.filter_pipeline(x, o, kinds[kind], param)
    torch.cuda.synchronize()
    assert p.last_launch_count() == 3 * batch
    H = filt_H(kind, N, M, param)
    ref = np.stack([oracle.filter_pipeline_real(imgs[i], H)[0] for i in range(batch)])
    assert oracle.rel_l2(o.cpu().numpy(), ref) <= 1e-5
    p.destroy()


def test_half_spectrum_pipeline_8192(b):
    """The real-to-real Gaussian pipeline at the C4 size (8192^2): beyond the
    real-pair passes' 2048 limit, so through the half spectrum."""
    N = M = 8192
    img = fixtures.sky_image(N, M, seed=1950, nsrc=2000)
    p = b.Plan((N, M), batch=1, flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    x = torch.from_numpy(img).cuda()
    o = torch.empty_like(x)
    p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    ref, im = oracle.filter_pipeline_real(img, oracle.gauss_filter(N, M, 0.1))
    assert oracle.rel_l2(o.cpu().numpy(), ref) <= 1e-5
    p.destroy()


def test_real_entry_point_errors(b):
    p = b.Plan((1,), batch=1)
    x = torch.zeros(4, dtype=torch.float32, device="cuda")
    h = torch.zeros(4, dtype=torch.complex64, device="cuda")
    with pytest.raises(b.FFTError) as ei:
        p.forward_r2c(x, h)  # n = 1
    assert ei.value.status == 1
    q = b.Plan((8, 8), batch=1)
    with pytest.raises(b.FFTError) as ei:
        q.forward_r2c(x, x)  # in place
    assert ei.value.status == 2


@pytest.mark.parametrize("cols1", ["1", "0"])
@pytest.mark.parametrize("M,batch", [(256, 2), (2048, 1), (32, 1)])
def test_half_spectrum_pipeline_8192_rows_colfilt(b, M, batch, cols1, monkeypatch):
    """8192-row real-to-real Gaussian pipelines: the half spectrum padded to
    M/2 + 16 bins per row and filtered by the one-pass k_colfilt (g_N(u) g_M(v)
    / (N M)), or (B200FFT_PIPE_COLS1=0) unpadded through k_cols, both against
    the oracle."""
    monkeypatch.setenv("B200FFT_PIPE_COLS1", cols1)
    N = 8192
    imgs = np.stack([fixtures.sky_image(N, M, seed=1960 + i, nsrc=200) for i in range(batch)])
    p = b.Plan((N, M), batch=batch, flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty_like(x)
    p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    assert p.last_launch_count() == 3 * batch
    H = oracle.gauss_filter(N, M, 0.1)
    ref = np.stack([oracle.filter_pipeline_real(imgs[i], H)[0] for i in range(batch)])
    assert oracle.rel_l2(o.cpu().numpy(), ref) <= 1e-5
    p.destroy()
