"""Pins of the real-input (half-spectrum) oracle functions:
independent library routines (numpy's pocketfft rfft / irfft), closed forms
and round trips -- none of them re-derives the oracle's own formula."""
import numpy as np
import pytest

import oracle

RNG = np.random.default_rng(20261020)

SHAPES = [(1, 2), (2, 2), (4, 8), (8, 4), (16, 64), (64, 32), (256, 256)]


@pytest.mark.parametrize("N,M", SHAPES)
def test_rfft2d_matches_pocketfft(N, M):
    f = RNG.standard_normal((N, M))
    got = oracle.rfft2d(f)
    assert got.shape == (N, M // 2 + 1)
    ref = np.fft.rfft2(f) / N  # eq5's 1/N (N = rows)
    assert np.max(np.abs(got - ref)) <= 1e-13 * max(1.0, np.max(np.abs(ref)))


@pytest.mark.parametrize("N,M", SHAPES)
def test_irfft2d_matches_pocketfft_and_round_trips(N, M):
    f = RNG.standard_normal((N, M))
    F = oracle.rfft2d(f)
    g, im = oracle.irfft2d(F, M)
    assert im <= 1e-13 * max(1.0, np.max(np.abs(f)))
    assert np.max(np.abs(g - f)) <= 1e-13 * max(1.0, np.max(np.abs(f)))  # C2R o R2C = id
    # 2D-IDFT with 1/M = numpy's irfft2 (1/(N M)) times N
    G = RNG.standard_normal((N, M // 2 + 1)) + 1j * RNG.standard_normal((N, M // 2 + 1))
    G = oracle.rfft2d(np.fft.irfft2(G, s=(N, M)))  # a consistent Hermitian half spectrum
    g2, _ = oracle.irfft2d(G, M)
    assert np.max(np.abs(g2 - np.fft.irfft2(G, s=(N, M)) * N)) <= 1e-12 * max(1.0, np.max(np.abs(g2)))


def test_real_closed_forms():
    N, M = 8, 16
    c = np.full((N, M), 2.5)
    F = oracle.rfft2d(c)
    exp = np.zeros((N, M // 2 + 1), complex)
    exp[0, 0] = M * 2.5  # eq5: (1/N) * N M c
    assert np.max(np.abs(F - exp)) <= 1e-13
    d = np.zeros((N, M))
    d[0, 0] = 1.0
    assert np.max(np.abs(oracle.rfft2d(d) - 1.0 / N)) <= 1e-15  # flat 1/N
    # Hermitian extension: the full spectrum of a real image equals fft2d's
    f = RNG.standard_normal((N, M))
    full = oracle.hermitian_extend(oracle.rfft2d(f), M)
    assert np.max(np.abs(full - oracle.fft2d(f.astype(complex)))) <= 1e-13


@pytest.mark.parametrize("n", [2, 4, 16, 1024])
def test_rfft_batch_1d(n):
    x = RNG.standard_normal((3, n))
    got = oracle.rfft_batch(x)
    assert np.max(np.abs(got - np.fft.rfft(x, axis=-1) / n)) <= 1e-13
    back, im = oracle.irfft_batch(got, n)
    assert im <= 1e-13 and np.max(np.abs(back - x)) <= 1e-12  # Sec. 3 inverse of Eq. E2 = identity
    c = RNG.standard_normal((3, n // 2 + 1)) + 1j * RNG.standard_normal((3, n // 2 + 1))
    c[:, 0] = c[:, 0].real
    if n >= 2:
        c[:, -1] = c[:, -1].real
    g, _ = oracle.irfft_batch(c, n)
    assert np.max(np.abs(g - np.fft.irfft(c, n, axis=-1) * n)) <= 1e-12 * max(1.0, np.max(np.abs(g)))


@pytest.mark.parametrize("kind", ["gauss", "literal", "lowpass"])
def test_filter_pipeline_real_is_the_complex_pipeline(kind):
    """For a real image and a real H with H(u, v) = H(-u, -v) -- the Gaussian
    and both readings of Eq. (filtro) -- the pipeline through the half
    spectrum equals the complex pipeline, whose imaginary part vanishes."""
    N, M = 64, 128
    f = RNG.uniform(0, 255, (N, M))
    if kind == "gauss":
        H = oracle.gauss_filter(N, M, 0.1)
    else:
        H = oracle.ideal_filter(N, M, 20.0 if kind == "lowpass" else 40.0, literal=(kind == "literal"))
    u = (-np.arange(N)) % N
    v = (-np.arange(M)) % M
    assert np.array_equal(H, H[u][:, v])  # the symmetry the half-spectrum path needs
    got, im = oracle.filter_pipeline_real(f, H)
    ref = oracle.filter_pipeline(f.astype(complex), H)
    assert np.max(np.abs(ref.imag)) <= 1e-12 * np.max(np.abs(ref.real))
    assert np.max(np.abs(got - ref.real)) <= 1e-12 * np.max(np.abs(ref.real))
    assert im <= 1e-12 * np.max(np.abs(ref.real))
