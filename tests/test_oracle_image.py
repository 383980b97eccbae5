"""Pins of the oracle's image application (Sec. 6; SURVEY
NEXT-1) against facts the paper and arithmetic fix, independent of the
oracle's own formulas (CPU only)."""
import math

import numpy as np
import pytest

import fixtures
import oracle


@pytest.mark.parametrize("shape,padded", [((506, 460), (512, 512)), ((3, 5), (4, 8)),
                                          ((512, 512), (512, 512)), ((1, 1), (1, 1)), ((33, 17), (64, 32))])
def test_pad_pow2_shapes(shape, padded):
    """P:366-367 "pads with zeros ... to complete the next power of two";
    the paper's 460 x 506 photograph becomes 512 x 512."""
    rng = np.random.default_rng(1)
    img = rng.integers(0, 256, size=shape).astype(np.uint8)
    g = oracle.pad_pow2(img)
    assert g.shape == padded
    assert np.array_equal(g[: shape[0], : shape[1]].real, img.astype(np.float64))
    mask = np.ones(padded, bool)
    mask[: shape[0], : shape[1]] = False
    assert not np.any(g[mask]) and not np.any(g.imag)


def test_spectrum_values():
    """|3 + 4i| = 5; the spectrum of the constant-ones grid under
    eq5's 1/N is M at (0, 0) and 0 elsewhere (sum of N M ones / N)."""
    assert oracle.spectrum(np.array([3 + 4j]))[0] == 5.0
    N, M = 8, 16
    s = oracle.spectrum(oracle.fft2d(np.ones((N, M))))
    assert abs(s[0, 0] - M) < 1e-12
    s[0, 0] = 0
    assert s.max() < 1e-12


def lattice_count(b, N, M):
    """Integer points (k_u, k_v) in [-N/2, N/2) x [-M/2, M/2) with k_u^2 +
    k_v^2 <= b^2, counted column by column with integer square roots."""
    b2 = int(round(b * b))
    n = 0
    for ku in range(-N // 2, N // 2):
        r = b2 - ku * ku
        if r < 0:
            continue
        t = math.isqrt(r)
        n += min(t, M // 2 - 1) + min(t, M // 2) + 1
    return n


@pytest.mark.parametrize("N,M,b", [(512, 512, 340.0), (64, 32, 10.0), (8, 8, 0.0)])
def test_ideal_filter_lattice_counts(N, M, b):
    """Eq. (filtro) with b = 340 on the paper's padded 512^2 grid:
    the low-pass reading keeps exactly the lattice points within radius b of
    the zero frequency; the literal reading zeroes exactly as many points
    around (N/2, M/2) (same lattice, shifted)."""
    n = lattice_count(b, N, M)
    low = oracle.ideal_filter(N, M, b, literal=False)
    lit = oracle.ideal_filter(N, M, b, literal=True)
    assert int(low.sum()) == n
    assert int((lit == 0).sum()) == n
    assert set(np.unique(low)) <= {0.0, 1.0} and set(np.unique(lit)) <= {0.0, 1.0}
    if b == 0.0:  # only the distance-0 point: the centre (literal), DC (low-pass)
        assert lit[N // 2, M // 2] == 0 and int((lit == 0).sum()) == 1
        assert low[0, 0] == 1 and int(low.sum()) == 1


def test_image_allpass_identity():
    """H = 1 (and a low-pass disk covering the whole padded grid): the
    pipeline is the identity up to fp64 rounding, so the rounded, cropped
    output reproduces the 8-bit input exactly (SPEC's +-1 bound, tightened)."""
    img = fixtures.sky_image_u8(50, 37, seed=11, nsrc=10)
    for filt, b in (("none", 0.0), ("lowpass", 1e6)):
        r = oracle.image_filter_u8(img, filt, b)
        assert (r["N"], r["M"]) == (64, 64)
        assert r["u8"].shape == img.shape
        assert np.array_equal(r["u8"], img)
        assert np.abs(r["real"] - img).max() < 1e-9


def test_image_uniform_keeps_dc():
    """A uniform image on a power-of-two grid has all its energy at DC, which
    every low-pass disk with b >= 0 keeps: output = input."""
    img = np.full((64, 64), 173, np.uint8)
    r = oracle.image_filter_u8(img, "lowpass", 1.0)
    assert np.array_equal(r["u8"], img)


def test_image_clamp_and_round():
    """Clamp to [0, max_val] after rounding: with H = 1 and max_val = 200 the
    output is min(img, 200) exactly; with an all-zero filter (literal disk
    covering the grid) the output is 0 everywhere."""
    img = np.arange(64 * 16, dtype=np.int64).reshape(64, 16) % 256
    img = img.astype(np.uint8)
    r = oracle.image_filter_u8(img, "none", 0.0, max_val=200)
    assert np.array_equal(r["u8"], np.minimum(img, 200))
    r = oracle.image_filter_u8(img, "literal", 1e6)
    assert not np.any(r["u8"]) and np.abs(r["real"]).max() < 1e-9


def test_image_energy_monotone():
    """Narrower low-pass disks keep less spectral energy: b = 8 < 16 < 32.
    Parseval with eq5's 1/N and the 2D-IDFT's 1/M on a square grid
    (sum |f|^2 = (N/M) sum |F|^2 = sum |F|^2) ties the filtered image's
    energy to the kept spectral energy (the disk is symmetric under k -> -k,
    so the filtered image of a real image is real)."""
    img = fixtures.sky_image_u8(64, 64, seed=12, nsrc=20)
    e = []
    for b in (8.0, 16.0, 32.0):
        r = oracle.image_filter_u8(img, "lowpass", b)
        H = oracle.ideal_filter(64, 64, b, literal=False)
        kept = float(np.sum((r["spectrum"] * H) ** 2))
        assert abs(float(np.sum(r["real"] ** 2)) - kept) <= 1e-9 * kept
        e.append(kept)
    assert e[0] < e[1] < e[2]


@pytest.mark.parametrize("N,M", [(64, 64), (32, 128)])
def test_real_gauss_pipeline_stays_real(N, M):
    """NEXT-3's premise (R19): for a real image and the real, even
    Gaussian H, the pipeline preserves Hermitian symmetry, so its output is
    real -- the imaginary part of the oracle's complex result vanishes to
    fp64 rounding -- and equals the separable row-then-column application of
    the 1D operators (rows filtered, then columns) on real data."""
    img = fixtures.sky_image(N, M, seed=21, nsrc=10).astype(np.float64)
    out = oracle.gauss_pipeline(img.astype(np.complex128), 0.1)
    assert np.abs(out.imag).max() <= 1e-12 * np.abs(out.real).max()
    H = oracle.gauss_filter(N, M, 0.1)
    g_v = H[0] / H[0, 0]  # row factor g_M(v): H(0, v) = g_N(0) g_M(v), g_N(0) = 1
    g_u = H[:, 0] / H[0, 0]
    rows = np.real(np.fft.ifft(np.fft.fft(img, axis=1) * g_v[None, :], axis=1))
    both = np.real(np.fft.ifft(np.fft.fft(rows, axis=0) * g_u[:, None], axis=0))
    assert oracle.rel_l2(out.real, both) <= 1e-12
