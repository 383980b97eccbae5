"""fp64 CPU oracle for arXiv cs/0103001 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product library (``paper_cs_0103001_b200``) never imports, links or calls it
and shares no code with it.

Thin ctypes wrapper over ``oracle.c``; every function there cites the PAPER.md
passage it follows.  Arrays are numpy complex128 (interleaved re/im doubles).
All functions are pinned by ``tests/test_oracle.py`` (nothing here is "parity
unpinned").
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile oracle.c (gcc -O2 -fopenmp, no fast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-fno-fast-math",
             "-o", _SO, src, "-lm"]
        )
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, vp, ci, cd = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        sig = {
            "oracle_bitrev_order": [i64, vp],
            "oracle_fft": [vp, vp, i64],
            "oracle_ifft": [vp, vp, i64],
            "oracle_ifft_plus_tree": [vp, vp, i64],
            "oracle_dft_bruteforce": [vp, vp, i64, ci],
            "oracle_eval_exp_poly": [vp, i64, cd, vp],
            "oracle_fft_batch": [vp, vp, i64, i64, ci],
            "oracle_fft2d": [vp, vp, i64, i64],
            "oracle_ifft2d": [vp, vp, i64, i64],
            "oracle_dft2d_bruteforce": [vp, vp, i64, i64, ci],
            "oracle_gauss_filter": [i64, i64, cd, vp],
            "oracle_filter_pipeline": [vp, vp, i64, i64, vp],
            "oracle_gauss_pipeline": [vp, vp, i64, i64, cd],
            "oracle_dft_bins": [vp, i64, vp, i64, ci, vp],
            "oracle_dft_bins_c64": [vp, i64, vp, i64, ci, vp],
        }
        for name, args in sig.items():
            f = getattr(lib, name)
            f.argtypes = args
            f.restype = ci
        lib.oracle_num_threads.restype = ci
        lib.oracle_set_num_threads.argtypes = [ci]
        _lib = lib
    return _lib


def _c128(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.complex128))


def _check(rc: int, what: str):
    if rc != 0:
        raise OracleError(f"{what}: oracle status {rc}")


def num_threads() -> int:
    return _load().oracle_num_threads()


def set_num_threads(t: int) -> None:
    _load().oracle_set_num_threads(int(t))


def bitrev_order(n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    _check(_load().oracle_bitrev_order(n, out.ctypes.data), "bitrev_order")
    return out


def fft(x) -> np.ndarray:
    """Eq. E2: (1/N) sum_j x_j e^{-2 pi i jk/N} via the paper's tree (O2)."""
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_fft(x.ctypes.data, out.ctypes.data, x.size), "fft")
    return out


def ifft(c) -> np.ndarray:
    """Sec. 3 inverse: N * FFT(c)[(N-k) mod N], unscaled +sign sum (O3)."""
    c = _c128(c)
    out = np.empty_like(c)
    _check(_load().oracle_ifft(c.ctypes.data, out.ctypes.data, c.size), "ifft")
    return out


def ifft_plus_tree(c) -> np.ndarray:
    c = _c128(c)
    out = np.empty_like(c)
    _check(_load().oracle_ifft_plus_tree(c.ctypes.data, out.ctypes.data, c.size), "ifft_plus")
    return out


def dft_bruteforce(x, inverse: bool = False) -> np.ndarray:
    x = _c128(x)
    out = np.empty_like(x)
    _check(_load().oracle_dft_bruteforce(x.ctypes.data, out.ctypes.data, x.size, int(inverse)),
           "dft_bruteforce")
    return out


def eval_exp_poly(c, x: float) -> complex:
    c = _c128(c)
    out = np.empty(1, dtype=np.complex128)
    _check(_load().oracle_eval_exp_poly(c.ctypes.data, c.size, float(x), out.ctypes.data),
           "eval_exp_poly")
    return complex(out[0])


def fft_batch(x, inverse: bool = False) -> np.ndarray:
    """Rows of a 2D array transformed independently (OpenMP over rows)."""
    x = _c128(x)
    assert x.ndim == 2
    out = np.empty_like(x)
    _check(_load().oracle_fft_batch(x.ctypes.data, out.ctypes.data, x.shape[1], x.shape[0],
                                    int(inverse)), "fft_batch")
    return out


def fft2d(f) -> np.ndarray:
    """eq5 (1/N, N = rows) via rows -> x M -> columns (O4)."""
    f = _c128(f)
    out = np.empty_like(f)
    _check(_load().oracle_fft2d(f.ctypes.data, out.ctypes.data, *f.shape), "fft2d")
    return out


def ifft2d(F) -> np.ndarray:
    """2D-IDFT (1/M, M = columns) (O4)."""
    F = _c128(F)
    out = np.empty_like(F)
    _check(_load().oracle_ifft2d(F.ctypes.data, out.ctypes.data, *F.shape), "ifft2d")
    return out


def dft2d_bruteforce(f, inverse: bool = False) -> np.ndarray:
    f = _c128(f)
    out = np.empty_like(f)
    _check(_load().oracle_dft2d_bruteforce(f.ctypes.data, out.ctypes.data, f.shape[0],
                                           f.shape[1], int(inverse)), "dft2d_bruteforce")
    return out


def gauss_filter(N: int, M: int, param: float = 0.1) -> np.ndarray:
    H = np.empty((N, M), dtype=np.float64)
    _check(_load().oracle_gauss_filter(N, M, float(param), H.ctypes.data), "gauss_filter")
    return H


def filter_pipeline(f, H) -> np.ndarray:
    f = _c128(f)
    H = np.ascontiguousarray(H, dtype=np.float64)
    out = np.empty_like(f)
    _check(_load().oracle_filter_pipeline(f.ctypes.data, out.ctypes.data, f.shape[0], f.shape[1],
                                          H.ctypes.data), "filter_pipeline")
    return out


def gauss_pipeline(f, param: float = 0.1) -> np.ndarray:
    f = _c128(f)
    out = np.empty_like(f)
    _check(_load().oracle_gauss_pipeline(f.ctypes.data, out.ctypes.data, f.shape[0], f.shape[1],
                                         float(param)), "gauss_pipeline")
    return out


# ---- the paper's image application (Sec. 6) ----

def next_pow2(d: int) -> int:
    """Smallest power of two >= d (d >= 1)."""
    p = 1
    while p < d:
        p *= 2
    return p


def pad_pow2(img, N: int | None = None, M: int | None = None) -> np.ndarray:
    """"pads with zeros on rows and on columns to complete the next
    power of two": the image at the top-left of an N x M zero grid (default
    N, M = next powers of two of its height and width), as complex128."""
    img = np.asarray(img)
    h, w = img.shape
    N = next_pow2(h) if N is None else N
    M = next_pow2(w) if M is None else M
    g = np.zeros((N, M), dtype=np.complex128)
    g[:h, :w] = img.astype(np.float64)
    return g


def spectrum(F) -> np.ndarray:
    """sqrt(Re[C(x,y)]^2 + Im[C(x,y)]^2), elementwise."""
    F = np.asarray(F, dtype=np.complex128)
    return np.sqrt(F.real * F.real + F.imag * F.imag)


def ideal_filter(N: int, M: int, b: float, literal: bool = True) -> np.ndarray:
    """Eq. (filtro), evaluated per (u, v) in fp64.  literal
    (R13): F = 0 if sqrt((u - N/2)^2 + (v - M/2)^2) <= b, else 1, on
    the unshifted spectrum, (c1, c2) = (N/2, M/2) the grid's centre.
    literal=False: the centred low-pass reading, 1 if sqrt(k_u^2 + k_v^2) <= b
    with signed indices k_u = u (u < N/2) else u - N, else 0."""
    H = np.empty((N, M), dtype=np.float64)
    for u in range(N):
        if literal:
            d2 = (u - N // 2) ** 2 + (np.arange(M) - M // 2) ** 2
            H[u] = np.where(np.sqrt(d2) <= b, 0.0, 1.0)
        else:
            ku = u if u < N // 2 else u - N
            kv = np.where(np.arange(M) < M // 2, np.arange(M), np.arange(M) - M)
            H[u] = np.where(np.sqrt(ku * ku + kv * kv) <= b, 1.0, 0.0)
    return H


def image_filter_u8(img, filt: str = "literal", param: float = 340.0, max_val: int = 255,
                    N: int | None = None, M: int | None = None) -> dict:
    """Sec. 6 end to end, in the paper's order: pad to powers of
    two -> 2D FFT (eq5, O4) -> spectrum -> multiply Re and Im by
    the filter -> 2D-IFFT (O4) -> real part -> round
    half up -> clamp to [0, max_val] -> crop to the original h x w (the
    digital image of P:356-361).  filt: "literal" / "lowpass" (Eq. filtro,
    b = param) or "gauss" (O5 with param x Nyquist).  Returns the padded grid
    size, the spectrum, the real part before rounding (cropped) and the uint8
    image."""
    img = np.asarray(img)
    h, w = img.shape
    g = pad_pow2(img, N, M)
    N, M = g.shape
    F = fft2d(g)
    spec = spectrum(F)
    if filt == "gauss":
        H = gauss_filter(N, M, param)
    elif filt in ("literal", "lowpass"):
        H = ideal_filter(N, M, param, literal=(filt == "literal"))
    elif filt == "none":
        H = np.ones((N, M))
    else:
        raise ValueError(filt)
    f = ifft2d(F * H)
    real = f.real[:h, :w].copy()
    out = np.clip(np.floor(real + 0.5), 0, max_val).astype(np.uint8)
    return {"N": N, "M": M, "spectrum": spec, "real": real, "u8": out}


# ---- the paper's parallel schedule (Sec. 4) ----

def paper_tree_fft(x, P: int) -> np.ndarray:
    """The paper's parallel FFT, step by step, fp64: processor q
    of P = 2^l transforms its branch, the cyclic subsequence x[q + P j]
    (with this oracle's O2 and its 1/len); then while nproc_sup
    = S > 1, processor q + S/2 hands its vector to q, which
    combines them with one radix-2 level, Y[k] = (E[k] + w^k O[k]) / 2,
    Y[k + M] = (E[k] - w^k O[k]) / 2 with w = exp(-2 pi i / (2M)) (the
    paper's Z factors, Table 2, and its 1/N); the MASTER ends with X."""
    x = np.asarray(x, dtype=np.complex128).ravel()
    n = x.size
    assert P >= 1 and P & (P - 1) == 0 and n % P == 0
    vec = [fft(x[q::P]) for q in range(P)]
    S = P
    while S > 1:
        M = vec[0].size
        k = np.arange(M)
        w = np.exp(-2j * np.pi * k / (2 * M))
        for q in range(S // 2):
            E, O = vec[q], vec[q + S // 2]
            vec[q] = np.concatenate([(E + w * O) / 2, (E - w * O) / 2])
        S //= 2
    return vec[0]


def paper_parallel_products(m: int, l: int) -> int:
    """Eq. (multi): complex products of the parallel FFT with
    N = 2^m data on 2^l processors, (m - l) 2^(m - l) + sum_{i=1..l} 2^(m-l+i)."""
    return (m - l) * 2 ** (m - l) + sum(2 ** (m - l + i) for i in range(1, l + 1))


# ---- real input, half spectrum (R2C / C2R) -----------------
# The paper's images are real, integer-valued rasters (Sec. 6).
# For real f the DFT is Hermitian, F(u, v) = conj F(-u mod N, -v mod M), so
# the columns v = 0 .. M/2 determine it; these functions are the paper's
# transforms (eq5; 2D-IDFT; Eq. E2 / Sec. 3 in 1D)
# written through that symmetry, on top of the pinned O2 / O4 above.

def hermitian_extend(half, M: int) -> np.ndarray:
    """[..., N, M/2 + 1] half spectrum -> the full [..., N, M] spectrum of a
    real signal: F(u, v) for v > M/2 is conj F((N - u) mod N, M - v).  1D:
    pass a [..., M/2 + 1] array with a trailing axis only (N absent)."""
    half = np.asarray(half, dtype=np.complex128)
    h = M // 2 + 1
    assert half.shape[-1] == h
    full = np.zeros(half.shape[:-1] + (M,), dtype=np.complex128)
    full[..., :h] = half
    v = np.arange(h, M)
    if half.ndim >= 2:
        N = half.shape[-2]
        u = np.arange(N)
        full[..., :, h:] = np.conj(half[..., (-u) % N, :][..., :, M - v])
    else:
        full[..., h:] = np.conj(half[..., M - v])
    return full


def rfft2d(f) -> np.ndarray:
    """eq5 of a real N x M image (promoted exactly), columns v = 0 .. M/2."""
    f = np.asarray(f)
    M = f.shape[-1]
    return fft2d(f.astype(np.complex128))[:, : M // 2 + 1]


def irfft2d(half, M: int):
    """2D-IDFT (1/M) of the Hermitian spectrum whose columns 0 .. M/2 are
    `half`; returns (real part, max |imaginary part|) -- the latter ~1e-16
    relative for a consistent half spectrum."""
    g = ifft2d(hermitian_extend(half, M))
    return g.real.copy(), float(np.max(np.abs(g.imag))) if g.size else 0.0


def rfft_batch(x) -> np.ndarray:
    """Eq. E2 (1/n) of each real row, bins k = 0 .. n/2."""
    x = np.asarray(x)
    n = x.shape[-1]
    return fft_batch(x.astype(np.complex128).reshape(-1, n))[:, : n // 2 + 1].reshape(x.shape[:-1] + (n // 2 + 1,))


def irfft_batch(half, n: int):
    """Sec. 3 inverse (unscaled) of each Hermitian row given by bins 0 .. n/2;
    returns (real part, max |imaginary part|)."""
    half = np.asarray(half, dtype=np.complex128)
    rows = half.reshape(-1, n // 2 + 1)
    full = np.stack([hermitian_extend(r, n) for r in rows])  # 1D extension, row by row
    g = fft_batch(full, inverse=True).reshape(half.shape[:-1] + (n,))
    return g.real.copy(), float(np.max(np.abs(g.imag))) if g.size else 0.0


def filter_pipeline_real(f, H):
    """Sec. 6's pipeline on a real image through the half spectrum:
    2D-IDFT(H .* eq5(f)) with H real and H(u, v) = H(-u, -v) (the Gaussian
    and both readings of Eq. filtro), so the result is real; returns (real
    output, max |imaginary part| of the full complex pipeline)."""
    f = np.asarray(f)
    M = f.shape[-1]
    half = rfft2d(f) * np.asarray(H, dtype=np.float64)[:, : M // 2 + 1]
    return irfft2d(half, M)


def dft_bins(x, bins, inverse: bool = False) -> np.ndarray:
    """Selected bins of one transform by compensated direct sums (O7)."""
    bins = np.ascontiguousarray(bins, dtype=np.int64)
    out = np.empty(bins.size, dtype=np.complex128)
    if isinstance(x, np.ndarray) and x.dtype == np.complex64 and x.flags.c_contiguous:
        fn = _load().oracle_dft_bins_c64  # exact promotion inside, no 16 GiB copy at 2^30
    else:
        x = _c128(x)
        fn = _load().oracle_dft_bins
    _check(fn(x.ctypes.data, x.size, bins.ctypes.data, bins.size, int(inverse), out.ctypes.data),
           "dft_bins")
    return out


def rel_l2(a, ref) -> float:
    """O8: sqrt(sum |a-ref|^2) / sqrt(sum |ref|^2), fp64 (numpy pairwise sums)."""
    a = np.asarray(a).astype(np.complex128, copy=False).ravel()
    ref = np.asarray(ref).astype(np.complex128, copy=False).ravel()
    d = a - ref
    num = np.sum(d.real * d.real + d.imag * d.imag)
    den = np.sum(ref.real * ref.real + ref.imag * ref.imag)
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))
