"""Pins of the fp64 oracle against what the paper and the mathematics fix.

None of these compares the oracle with itself: every check is against a
closed form, an invariant, a brute-force definition, an independent library
routine (numpy's pocketfft), an FFT-free spatial computation, or a value the
paper prints (tests/golden/).  A plausible mistake anywhere in oracle.c (a
dropped term, a wrong sign or index, a transposed operand, a misplaced 1/N)
fails at least one of them.
"""
import numpy as np
import pytest

import fixtures
import oracle
from golden_util import read_golden

RNG = np.random.default_rng(20010301)


def rnd(n, rng=RNG):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def parse_vec(s):
    return np.array([complex(float(a), float(b)) for a, b in (p.split(",") for p in s.split(";"))])


# ---------------------------------------------------------------- tree leaves
def test_tree_leaf_order_matches_paper():
    # P:120-134 / P:179-190: leaves P_0 P_4 P_2 P_6 P_1 P_5 P_3 P_7
    golden = [int(v) for v in read_golden("tree_leaves_n8.txt")[0].split()]
    assert oracle.bitrev_order(8).tolist() == golden
    assert oracle.bitrev_order(2).tolist() == [0, 1]
    assert oracle.bitrev_order(4).tolist() == [0, 2, 1, 3]


@pytest.mark.parametrize("m", range(0, 13))
def test_bitrev_is_involution(m):
    p = oracle.bitrev_order(1 << m)
    assert np.array_equal(p[p], np.arange(1 << m))


# --------------------------------------------------- brute-force definition O9
@pytest.mark.parametrize("N", [1, 2, 3, 5, 8, 12, 17, 64])
def test_bruteforce_closed_forms(N):
    # impulse at j0 -> (1/N) e^{-2 pi i k j0 / N};  tone k0 -> delta_{k,k0}  (Eq. E2)
    k = np.arange(N)
    for j0 in {0, 1 % N, N - 1}:
        x = np.zeros(N, complex)
        x[j0] = 1
        exp = np.exp(-2j * np.pi * k * j0 / N) / N
        assert np.max(np.abs(oracle.dft_bruteforce(x) - exp)) < 1e-14
    for k0 in {0, N // 2, N - 1}:
        x = np.exp(2j * np.pi * k0 * k / N)
        X = oracle.dft_bruteforce(x)
        d = np.zeros(N)
        d[k0] = 1
        assert np.max(np.abs(X - d)) < 1e-14
    # inverse brute force = the unscaled + sign sum, Eq. E3 at x_k = 2 pi k / N
    c = rnd(N)
    ref = np.array([np.sum(c * np.exp(1j * np.arange(N) * 2 * np.pi * kk / N)) for kk in k])
    assert oracle.rel_l2(oracle.dft_bruteforce(c, inverse=True), ref) < 1e-13


# ------------------------------------------------------------- forward FFT O2
@pytest.mark.parametrize("m", range(0, 9))
def test_fft_matches_bruteforce(m):
    N = 1 << m
    for _ in range(20):
        x = rnd(N)
        assert oracle.rel_l2(oracle.fft(x), oracle.dft_bruteforce(x)) < 1e-13


def test_spec_golden_examples():
    for row in read_golden("spec_examples.txt"):
        op, xin, xout = (s.strip() for s in row.split("|"))
        x, exp = parse_vec(xin), parse_vec(xout)
        got = oracle.fft(x) if op == "fft" else oracle.ifft(x)
        assert np.max(np.abs(got - exp)) < 1e-15, row


@pytest.mark.parametrize("m", [1, 3, 6, 10, 14])
def test_fft_closed_forms(m):
    N = 1 << m
    k = np.arange(N)
    # impulse -> flat 1/N, bit-exact (1/N is a power of two)
    x = np.zeros(N, complex)
    x[0] = 1
    X = oracle.fft(x)
    assert np.array_equal(X, np.full(N, 1.0 / N, complex))
    # shifted impulse
    j0 = N // 3 + 1 if N > 2 else N - 1
    x = np.zeros(N, complex)
    x[j0] = 1
    assert np.max(np.abs(oracle.fft(x) - np.exp(-2j * np.pi * ((k * j0) % N) / N) / N)) < 1e-15
    # constant a -> X_0 = a, others 0
    a = 0.7 - 0.3j
    X = oracle.fft(np.full(N, a))
    assert abs(X[0] - a) < 1e-15 and np.max(np.abs(X[1:]), initial=0) < 1e-15
    # single tone k0 -> delta_{k0}
    k0 = N // 2 - 1 if N > 2 else 1
    X = oracle.fft(np.exp(2j * np.pi * ((k0 * k) % N) / N))
    d = np.zeros(N)
    d[k0] = 1
    assert np.max(np.abs(X - d)) < 1e-13


@pytest.mark.parametrize("m", [4, 9, 13, 16])
def test_parseval_and_linearity(m):
    N = 1 << m
    x, y = rnd(N), rnd(N)
    X, Y = oracle.fft(x), oracle.fft(y)
    # Parseval with the paper's 1/N: sum|x|^2 = N sum|X|^2
    lhs, rhs = np.sum(np.abs(x) ** 2), N * np.sum(np.abs(X) ** 2)
    assert abs(lhs - rhs) / lhs < 1e-13
    al, be = 0.3 - 1.1j, -2.0 + 0.25j
    assert oracle.rel_l2(oracle.fft(al * x + be * y), al * X + be * Y) < 1e-13


@pytest.mark.parametrize("m", [10, 12, 15, 17, 20])
def test_fft_matches_numpy_pocketfft(m):
    N = 1 << m
    x = rnd(N)
    assert oracle.rel_l2(oracle.fft(x), np.fft.fft(x) / N) < 1e-13
    assert oracle.rel_l2(oracle.ifft(x), np.fft.ifft(x) * N) < 1e-13


def test_fft_batch_rows_independent():
    x = rnd(8 * 256).reshape(8, 256)
    Y = oracle.fft_batch(x)
    assert oracle.rel_l2(Y, np.fft.fft(x, axis=1) / 256) < 1e-13
    Z = oracle.fft_batch(x, inverse=True)
    assert oracle.rel_l2(Z, np.fft.ifft(x, axis=1) * 256) < 1e-13


# -------------------------------------------------------------- inverse O3
@pytest.mark.parametrize("m", [0, 1, 2, 5, 8, 12])
def test_inverse_round_trips(m):
    N = 1 << m
    x = rnd(N)
    assert oracle.rel_l2(oracle.ifft(oracle.fft(x)), x) < 1e-13
    assert oracle.rel_l2(oracle.fft(oracle.ifft(x)), x) < 1e-13
    # Sec. 3 reversal == independent + sign tree, == brute-force + sign sum
    assert oracle.rel_l2(oracle.ifft(x), oracle.ifft_plus_tree(x)) < 1e-15
    if N <= 256:
        assert oracle.rel_l2(oracle.ifft(x), oracle.dft_bruteforce(x, inverse=True)) < 1e-13


@pytest.mark.parametrize("N", [1, 2, 8, 32, 64])
def test_inverse_is_exp_polynomial(N):
    # Eq. E3: p(x_j) with x_j = 2 pi j / N interpolates f; the Sec. 3
    # identity p(2 pi - x_k) = N (1/N sum_j c_j e^{-i j x_k})
    f = rnd(N)
    c = oracle.fft(f)
    for j in range(N):
        assert abs(oracle.eval_exp_poly(c, 2 * np.pi * j / N) - f[j]) < 1e-12
    cc = rnd(N)
    Fc = oracle.fft(cc)
    for kk in range(N):
        assert abs(oracle.eval_exp_poly(cc, 2 * np.pi - 2 * np.pi * kk / N) - N * Fc[kk]) < 1e-12
    # delta_{k0} spectrum -> e^{+2 pi i j k0 / N}
    k0 = N // 2
    d = np.zeros(N, complex)
    d[k0] = 1
    assert np.max(np.abs(oracle.ifft(d) - np.exp(2j * np.pi * ((np.arange(N) * k0) % N) / N))) < 1e-14


def test_exp_poly_trivial():
    assert abs(oracle.eval_exp_poly([1, 0, 0, 0], 1.234) - 1) < 1e-15
    assert abs(oracle.eval_exp_poly([0, 1], np.pi) - (-1)) < 1e-15


# ------------------------------------------------------------------- 2D O4
@pytest.mark.parametrize("N", [1, 2, 4, 8])
@pytest.mark.parametrize("M", [1, 2, 4, 8])
def test_2d_matches_double_sum(N, M):
    f = rnd(N * M).reshape(N, M)
    F = oracle.fft2d(f)
    assert oracle.rel_l2(F, oracle.dft2d_bruteforce(f)) < 1e-13
    assert oracle.rel_l2(oracle.ifft2d(F), f) < 1e-13
    assert oracle.rel_l2(oracle.ifft2d(f), oracle.dft2d_bruteforce(f, inverse=True)) < 1e-13
    # numpy: eq5 = (M) * fft2 / (N M) = fft2 / N ; 2D-IDFT = (N M) ifft2 / M = N ifft2
    assert oracle.rel_l2(F, np.fft.fft2(f) / N) < 1e-13
    assert oracle.rel_l2(oracle.ifft2d(f), np.fft.ifft2(f) * N) < 1e-13


@pytest.mark.parametrize("N,M", [(16, 16), (32, 8), (4, 64)])
def test_2d_closed_forms(N, M):
    # constant 1 -> F(0,0) = M, others 0   (eq5 with 1/N, N rows)
    F = oracle.fft2d(np.ones((N, M)))
    exp = np.zeros((N, M))
    exp[0, 0] = M
    assert np.max(np.abs(F - exp)) < 1e-13
    # F = M delta(0,0) -> inverse is all ones (2D-IDFT with 1/M)
    assert np.max(np.abs(oracle.ifft2d(exp) - 1)) < 1e-13
    # separable f = g (x) h -> F(u,v) = M * ghat[u] * hhat[v] (ghat, hhat paper-normalised)
    g, h = rnd(N), rnd(M)
    F = oracle.fft2d(np.outer(g, h))
    assert oracle.rel_l2(F, M * np.outer(np.fft.fft(g) / N, np.fft.fft(h) / M)) < 1e-13
    # 2D Parseval: sum|F|^2 = (M/N) sum|f|^2
    f = rnd(N * M).reshape(N, M)
    F = oracle.fft2d(f)
    assert abs(np.sum(np.abs(F) ** 2) - M / N * np.sum(np.abs(f) ** 2)) / np.sum(np.abs(f) ** 2) < 1e-12
    # rows-first == columns-first (order of the separable sums)
    cols_first = np.stack([oracle.fft(f[:, v]) for v in range(M)], axis=1) * N
    cols_first = np.stack([oracle.fft(cols_first[u]) for u in range(N)], axis=0) * M / N
    assert oracle.rel_l2(F, cols_first) < 1e-13
    # single 2D tone e^{2 pi i (u0 x/N + v0 y/M)} -> M delta(u0, v0)
    u0, v0 = N // 2 - 1 if N > 2 else 0, 1
    x, y = np.meshgrid(np.arange(N), np.arange(M), indexing="ij")
    F = oracle.fft2d(np.exp(2j * np.pi * (u0 * x / N + v0 * y / M)))
    exp = np.zeros((N, M))
    exp[u0, v0] = M
    assert np.max(np.abs(F - exp)) < 1e-12


# --------------------------------------------------------- Gaussian + pipeline
def test_gauss_filter_values():
    N = 64
    H = oracle.gauss_filter(N, N, 0.1)
    assert H[0, 0] == 1.0
    # even in each signed frequency, so the unshifted mask is a low-pass
    assert np.array_equal(H[1:, :], H[:0:-1, :]) and np.array_equal(H[:, 1:], H[:, :0:-1])
    # at k = sigma_k (= 0.05 N = 3.2 -> not an integer); check k = Nyquist edge
    assert abs(H[N // 2, 0] - np.exp(-50.0)) < 1e-30
    assert H[1, 1] < 1 and H.max() == 1.0


def spatial_gauss_pipeline(f, sigma_px, radius=40):
    """FFT-free closed form: circular convolution with the sampled,
    periodised, sum-normalised Gaussian of width sigma_px, separable."""
    t = np.arange(-radius, radius + 1)
    w = np.exp(-(t.astype(np.float64) ** 2) / (2 * sigma_px * sigma_px))
    w /= w.sum()
    out = np.zeros_like(f)
    for ti, wi in zip(t, w):
        out += wi * np.roll(f, ti, axis=0)
    res = np.zeros_like(f)
    for ti, wi in zip(t, w):
        res += wi * np.roll(out, ti, axis=1)
    return res


@pytest.mark.parametrize("N,M", [(64, 64), (256, 256), (2048, 2048), (64, 256), (256, 64)])
def test_gauss_pipeline_equals_spatial_convolution(N, M):
    """SURVEY F3 / DESIGN.md R7: with sigma_k = 0.05 x (the axis length) per
    axis, the pipeline is a circular convolution with the same sampled
    Gaussian of sigma = 10/pi px along BOTH axes, whatever N and M.  The
    rectangular cases pin the N != M branch of oracle_gauss_filter: a
    swapped sigma_N / sigma_M (or sigma from the wrong axis length) gives a
    4x wider / narrower spatial kernel along one axis and fails by O(1)."""
    rows = read_golden("gauss_sigma.txt")
    sigma_px = float(rows[1].split()[1])
    assert abs(sigma_px - 10 / np.pi) < 1e-15
    if N == 2048:
        f = fixtures.sky_image(2048, 2048, seed=3).astype(np.complex128)  # the C3 input
    else:
        f = rnd(N * M).reshape(N, M)
    got = oracle.gauss_pipeline(f, 0.1)
    ref = spatial_gauss_pipeline(f, sigma_px)
    assert oracle.rel_l2(got, ref) < 1e-12


def test_pipeline_invariants():
    N, M = 32, 64
    H = oracle.gauss_filter(N, M, 0.1)
    f = rnd(N * M).reshape(N, M)
    # H == 1 -> identity
    assert oracle.rel_l2(oracle.filter_pipeline(f, np.ones((N, M))), f) < 1e-13
    # constant image passes unchanged (H(0,0) = 1); flux is conserved
    c = np.full((N, M), 3.5 + 0j)
    assert np.max(np.abs(oracle.filter_pipeline(c, H) - c)) < 1e-12
    out = oracle.filter_pipeline(f, H)
    assert abs(out.sum() - f.sum()) / abs(f.sum()) < 1e-12
    # single 2D tone -> H(u0, v0) * tone
    u0, v0 = 3, N - 5
    x, y = np.meshgrid(np.arange(N), np.arange(M), indexing="ij")
    tone = np.exp(2j * np.pi * (u0 * x / N + v0 * y / M))
    assert np.max(np.abs(oracle.filter_pipeline(tone, H) - H[u0, v0] * tone)) < 1e-13
    # real input stays real (H real and even)
    r = RNG.standard_normal((N, M)).astype(complex)
    assert np.max(np.abs(oracle.filter_pipeline(r, H).imag)) < 1e-13


# ----------------------------------------------------------- sampled bins O7
@pytest.mark.parametrize("m", [10, 16, 20])
def test_dft_bins_match_library(m):
    N = 1 << m
    x = rnd(N)
    bins = np.array([0, 1, 7, N // 2, N - 1, N // 3, 12345 % N])
    got = oracle.dft_bins(x, bins)
    ref = (np.fft.fft(x) / N)[bins]
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) < 1e-12
    x32 = x.astype(np.complex64)
    assert np.max(np.abs(oracle.dft_bins(x32, bins) - (np.fft.fft(x32.astype(complex)) / N)[bins])) < 1e-12
    goti = oracle.dft_bins(x, bins, inverse=True)
    refi = (np.fft.ifft(x) * N)[bins]
    assert np.max(np.abs(goti - refi)) / np.max(np.abs(refi)) < 1e-12


# ------------------------------------------------------------------ fixtures
def test_fixtures_counter_based():
    a = fixtures.complex_input(1000, fixtures.NORMAL, seed=2)
    b = fixtures.complex_input(400, fixtures.NORMAL, seed=2, offset=300)
    assert np.array_equal(a[300:700], b)
    u = fixtures.complex_input(200000, fixtures.UNIFORM, seed=4, dtype=np.complex128)
    assert np.all(np.abs(u.real) <= 1) and np.all(np.abs(u.imag) <= 1)
    assert abs(u.real.mean()) < 0.01 and abs(u.real.var() - 1 / 3) < 0.01
    n = fixtures.complex_input(200000, fixtures.NORMAL, seed=2, dtype=np.complex128)
    assert abs(n.imag.mean()) < 0.01 and abs(n.imag.var() - 1) < 0.02
    c = fixtures.complex_input(10, fixtures.NORMAL, seed=2, dtype=np.complex128)
    assert np.array_equal(c.astype(np.complex64), a[:10])
    assert not np.array_equal(fixtures.complex_input(10, 1, seed=3), a[:10])


def test_sky_image_recipe():
    img = fixtures.sky_image(256, 256, seed=3, nsrc=20)
    assert img.dtype == np.float32 and img.shape == (256, 256)
    med = np.median(img)
    assert 98 < med < 102  # background 100 + N(0, 5^2)
    assert img.max() > 150  # point sources present
