"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds no arithmetic of the method (no DFT, twiddle or filter):
only the counter-based random generator of ``gen.c`` (reading R11)
and the BASELINE.json workload recipes built from it.  Both the tests'
oracle calls and the GPU path draw their inputs here, so they see identical
values.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libfixtures.so")
_lib = None

UNIFORM = 0  # re, im i.i.d. U[-1, 1]
NORMAL = 1  # re, im i.i.d. N(0, 1) (Box-Muller)


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src, "-lm"]
        )
    return _SO


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, u64 = ctypes.c_int64, ctypes.c_uint64
        vp = ctypes.c_void_p
        lib.fixtures_complex_f64.argtypes = [u64, u64, ctypes.c_int, i64, i64, vp]
        lib.fixtures_complex_f32.argtypes = [u64, u64, ctypes.c_int, i64, i64, vp]
        lib.fixtures_sky_image.argtypes = [u64, i64, i64, i64, ctypes.c_double, vp]
        for f in (lib.fixtures_complex_f64, lib.fixtures_complex_f32, lib.fixtures_sky_image):
            f.restype = None
        _lib = lib
    return _lib


def complex_input(count: int, kind: int, seed: int, stream: int = 0, offset: int = 0,
                  dtype=np.complex64, out: np.ndarray | None = None) -> np.ndarray:
    """``count`` complex values (global element indices offset..offset+count-1)."""
    lib = _load()
    dtype = np.dtype(dtype)
    if out is None:
        out = np.empty(count, dtype=dtype)
    assert out.dtype == dtype and out.flags.c_contiguous and out.size == count
    fn = lib.fixtures_complex_f32 if dtype == np.complex64 else lib.fixtures_complex_f64
    fn(seed, stream, kind, offset, count, out.ctypes.data)
    return out


def sky_image(rows: int = 2048, cols: int = 2048, seed: int = 3, nsrc: int = 500,
              psf: float = 1.5) -> np.ndarray:
    """BASELINE configs[2] synthetic sky image, float32 [rows][cols]."""
    lib = _load()
    out = np.empty((rows, cols), dtype=np.float32)
    lib.fixtures_sky_image(seed, rows, cols, nsrc, psf, out.ctypes.data)
    return out


def sky_image_u8(rows: int = 506, cols: int = 460, seed: int = 6, nsrc: int = 120) -> np.ndarray:
    """8-bit stand-in for the paper's photograph (NGC5194, 460 x 506 pixels,
    P:395-398; the image itself is not available): the synthetic sky image
    above, square-root display stretch to [0, 255] (v = 255 sqrt((x - min) /
    (max - min))), rounded half up, uint8 [rows][cols].  Input recipe only."""
    x = sky_image(rows, cols, seed=seed, nsrc=nsrc).astype(np.float64)
    x -= x.min()
    top = x.max()
    v = 255.0 * np.sqrt(x / top) if top > 0 else x
    return np.clip(np.floor(v + 0.5), 0, 255).astype(np.uint8)


# BASELINE.json configs -> (shape, kind, seed); DESIGN.md section "Inputs".
CONFIGS = {
    "C1": dict(n=1024, batch=1, kind=UNIFORM, seed=1, dtype=np.complex128),
    "C2": dict(n=65536, batch=4096, kind=NORMAL, seed=2, dtype=np.complex64),
    "C3": dict(rows=2048, cols=2048, seed=3, param=0.1),
    "C4": dict(rows=8192, cols=8192, kind=UNIFORM, seed=4, param=0.1),
    "C5": dict(n=1 << 30, kind=NORMAL, seed=5, dtype=np.complex64),
}
