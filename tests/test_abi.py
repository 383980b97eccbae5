"""CPU-side checks of the C-ABI library: it builds, loads, exports every
symbol include/b200fft.h declares, and validates arguments synchronously
(no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

import pytest

import paper_cs_0103001_b200 as b
from paper_cs_0103001_b200 import _build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "b200fft.h")


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return b.load_library()


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_]+\*?\s+\*?\s*(fft\w+)\s*\(", text, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ("fft_plan_create", "fft_forward", "fft_inverse", "fft2d_filter_pipeline"):
        assert n in names
    assert sorted(names) == sorted(b.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_status_strings(lib):
    for code, name in b.STATUS.items():
        assert lib.fft_status_string(code).decode() == name


def test_build_info(lib):
    assert "sm_100a" in b.build_info()


@pytest.mark.parametrize("dims,rank", [((3,), 1), ((0,), 1), ((1 << 31,), 1), ((12, 16), 2),
                                       ((16384, 16), 2), ((16, 16384), 2)])
def test_invalid_sizes_rejected_without_gpu(lib, dims, rank):
    h = ctypes.c_void_p()
    arr = (ctypes.c_int64 * rank)(*dims)
    st = lib.fft_plan_create_ex(ctypes.byref(h), arr, rank, 1, b.C64, 0)
    assert st == 1, b.STATUS.get(st)  # FFT_E_INVALID_SIZE
    assert not h.value
    assert len(lib.fft_last_error()) > 0


def test_invalid_args_rejected_without_gpu(lib):
    h = ctypes.c_void_p()
    arr = (ctypes.c_int64 * 1)(64)
    assert lib.fft_plan_create_ex(ctypes.byref(h), arr, 3, 1, b.C64, 0) == 2  # bad rank
    assert lib.fft_plan_create_ex(ctypes.byref(h), arr, 1, 1, 7, 0) == 2  # bad precision
    assert lib.fft_plan_create_ex(ctypes.byref(h), arr, 1, 1, b.C64, 1 << 9) == 2  # bad flag
    assert lib.fft_plan_create_ex(ctypes.byref(h), arr, 1, -1, b.C64, 0) == 1  # negative batch
    assert lib.fft_plan_create_ex(ctypes.byref(h), arr, 1, 1, b.C64, b.IN_REAL_F32) == 2
    assert lib.fft_forward(None, None, None) == 2
    assert lib.fft_plan_destroy(None) == 0


def test_plan_creation_without_device_reports_cuda_error(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    arr = (ctypes.c_int64 * 1)(64)
    st = lib.fft_plan_create_ex(ctypes.byref(h), arr, 1, 1, b.C64, 0)
    assert st == 4  # FFT_E_CUDA: no silent CPU fallback
    assert not h.value


def test_product_package_does_not_reference_the_oracle():
    pkg = os.path.join(ROOT, "paper_cs_0103001_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "liboracle" not in text, f
                assert "oracle_" not in text, f
