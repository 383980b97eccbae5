"""GPU parity: rectangular and batched 2D grids (eq5 /
2D-IDFT with the literal asymmetric 1/N forward and 1/M inverse),
every 2D code path with batch > 1, against the oracle applied grid by grid."""
import numpy as np
import pytest

import fixtures
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = {np.complex64: 1e-5, np.complex128: 1e-12}


@pytest.fixture(scope="module")
def b():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_cs_0103001_b200 as m

    m.load_library()
    return m


def grids(batch, N, M, dtype, seed):
    return fixtures.complex_input(batch * N * M, fixtures.UNIFORM, seed=seed, dtype=dtype).reshape(batch, N, M)


@pytest.mark.parametrize("dtype", [np.complex64, np.complex128])
@pytest.mark.parametrize("batch,N,M", [(3, 64, 128), (2, 256, 32), (4, 16, 1024), (2, 512, 512), (5, 1, 8)])
def test_batched_forward_inverse(b, dtype, batch, N, M):
    f = grids(batch, N, M, dtype, 500 + N + M)
    p = b.Plan((N, M), batch=batch, precision=b.C64 if dtype == np.complex64 else b.C128)
    fd = torch.from_numpy(f).cuda()
    F = torch.empty_like(fd)
    g = torch.empty_like(fd)
    p.forward(fd, F)
    p.inverse(fd, g)
    torch.cuda.synchronize()
    p.destroy()
    F, g = F.cpu().numpy(), g.cpu().numpy()
    refF = np.stack([oracle.fft2d(f[i]) for i in range(batch)])
    refg = np.stack([oracle.ifft2d(f[i]) for i in range(batch)])
    assert oracle.rel_l2(F, refF) <= TOL[dtype]
    assert oracle.rel_l2(g, refg) <= TOL[dtype]
    for i in range(batch):  # every grid, not just the sum
        assert oracle.rel_l2(F[i], refF[i]) <= 4 * TOL[dtype]


@pytest.mark.parametrize("batch,N,M,real", [(3, 256, 1024, False), (2, 2048, 512, True), (2, 4096, 256, False),
                                            (3, 64, 32, True), (2, 8192, 256, False)])
def test_batched_gauss_pipeline(b, batch, N, M, real):
    """Each Gaussian schedule (transposed-store rows for sides <= 2048, rows +
    tiled transposes for longer sides, rows + fused columns for small grids)
    on a batch of rectangular grids; N != M exercises the per-axis sigma
    (R7) and the 1/N, 1/M split."""
    if real:
        f = np.stack([fixtures.sky_image(N, M, seed=600 + i, nsrc=40) for i in range(batch)])
    else:
        f = grids(batch, N, M, np.complex64, 610 + N)
    p = b.Plan((N, M), batch=batch, flags=b.IN_REAL_F32 if real else 0)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty((batch, N, M), dtype=torch.complex64, device="cuda")
    p.filter_pipeline(fd, od, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    p.destroy()
    out = od.cpu().numpy()
    ref = np.stack([oracle.gauss_pipeline(f[i].astype(np.complex128), 0.1) for i in range(batch)])
    assert oracle.rel_l2(out, ref) <= 1e-5


@pytest.mark.parametrize("literal", [True, False])
def test_batched_ideal_pipeline(b, literal):
    batch, N, M, rad = 3, 128, 256, 40.0
    f = grids(batch, N, M, np.complex64, 620)
    p = b.Plan((N, M), batch=batch)
    fd = torch.from_numpy(f).cuda()
    od = torch.empty_like(fd)
    p.filter_pipeline(fd, od, b.FILTER_IDEAL_LITERAL if literal else b.FILTER_IDEAL_LOWPASS, rad)
    torch.cuda.synchronize()
    p.destroy()
    H = oracle.ideal_filter(N, M, rad, literal=literal)
    ref = np.stack([oracle.filter_pipeline(f[i], H) for i in range(batch)])
    assert oracle.rel_l2(od.cpu().numpy(), ref) <= 1e-5


def test_batched_image_filter(b):
    """NEXT-1 on a batch of three 8-bit images (one launch triple each)."""
    imgs = np.stack([fixtures.sky_image_u8(90, 70, seed=630 + i, nsrc=15) for i in range(3)])
    p = b.Plan((128, 128), batch=3)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty_like(x)
    sp = torch.empty((3, 128, 128), dtype=torch.float32, device="cuda")
    p.image_filter_u8(x, o, b.FILTER_IDEAL_LOWPASS, 20.0, 255, sp)
    torch.cuda.synchronize()
    p.destroy()
    o, sp = o.cpu().numpy(), sp.cpu().numpy()
    for i in range(3):
        ref = oracle.image_filter_u8(imgs[i], "lowpass", 20.0, N=128, M=128)
        d = np.abs(o[i].astype(int) - ref["u8"].astype(int))
        frac = ref["real"] - np.floor(ref["real"])
        amb = np.abs(frac - 0.5) < 2e-3
        assert d[~amb].max(initial=0) == 0 and d.max() <= 1
        assert oracle.rel_l2(sp[i], ref["spectrum"]) <= 1e-5


@pytest.mark.parametrize("batch,N,M", [(1, 2048, 2048), (2, 256, 512), (3, 1024, 256), (1, 512, 2048)])
def test_real_to_real_gauss_pipeline(b, batch, N, M):
    """NEXT-3: FFT_IN_REAL_F32 | FFT_OUT_REAL_F32 -- two real rows per complex
    line in both passes; float32 output against the real part of the
    oracle's complex pipeline (whose imaginary part is ~0, pinned on CPU)."""
    imgs = np.stack([fixtures.sky_image(N, M, seed=700 + i, nsrc=60) for i in range(batch)])
    p = b.Plan((N, M), batch=batch, flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty_like(x)
    p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
    torch.cuda.synchronize()
    assert p.last_launch_count() == 2 * batch
    p.destroy()
    ref = np.stack([oracle.gauss_pipeline(imgs[i].astype(np.complex128), 0.1).real for i in range(batch)])
    assert oracle.rel_l2(o.cpu().numpy(), ref) <= 1e-5


def test_real_to_real_other_filters_use_the_half_spectrum(b):
    """Since NEXT-3's R2C / C2R: a real-output plan runs the ideal filters too
    (through the half spectrum: 3 launches), matching the oracle."""
    img = fixtures.sky_image(256, 256, seed=77, nsrc=20)
    p = b.Plan((256, 256), flags=b.IN_REAL_F32 | b.OUT_REAL_F32)
    x = torch.from_numpy(img).cuda()
    o = torch.empty_like(x)
    p.filter_pipeline(x, o, b.FILTER_IDEAL_LOWPASS, 10.0)
    torch.cuda.synchronize()
    assert p.last_launch_count() == 3
    ref, _ = oracle.filter_pipeline_real(img, oracle.ideal_filter(256, 256, 10.0, literal=False))
    assert oracle.rel_l2(o.cpu().numpy(), ref) <= 1e-5
    p.destroy()


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("real_out", [False, True])
@pytest.mark.parametrize("N,batch", [(512, 2), (1024, 3), (2048, 2)])
def test_fused_two_pass_pipeline(b, N, batch, real_out, fused, monkeypatch):
    """The square real-pair pipeline with both passes in one cooperative
    launch (k_rows_tma2, a grid barrier between the passes) against the
    two-launch form and the oracle; the plan is called twice so the barrier
    counter's later generations are exercised too."""
    monkeypatch.setenv("B200FFT_PIPE_FUSED2", fused)
    imgs = np.stack([fixtures.sky_image(N, N, seed=900 + i, nsrc=50) for i in range(batch)])
    flags = b.IN_REAL_F32 | (b.OUT_REAL_F32 if real_out else 0)
    p = b.Plan((N, N), batch=batch, flags=flags)
    x = torch.from_numpy(imgs).cuda()
    o = torch.empty((batch, N, N), dtype=torch.float32 if real_out else torch.complex64, device="cuda")
    for _ in range(2):
        o.zero_()
        p.filter_pipeline(x, o, b.FILTER_GAUSS, 0.1)
        torch.cuda.synchronize()
        assert p.last_launch_count() == (batch if fused == "1" and not real_out else 2 * batch)
        ref = np.stack([oracle.gauss_pipeline(imgs[i].astype(np.complex128), 0.1) for i in range(batch)])
        out = o.cpu().numpy()
        if real_out:
            assert oracle.rel_l2(out, ref.real) <= 1e-5
        else:
            assert oracle.rel_l2(out, ref) <= 1e-5
            assert np.all(out.imag == 0)
    p.destroy()
