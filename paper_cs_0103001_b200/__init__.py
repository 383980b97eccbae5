"""paper_cs_0103001_b200 -- Python binding of libb200fft (B200, sm_100a).

Argument marshalling only: every transform runs in the library's CUDA
kernels behind the C ABI of ``include/b200fft.h``.  There is no CPU or
library fallback: if ``lib/libb200fft.so`` is missing, importing the binding
raises.  PyTorch provides device memory and streams (plumbing only).

The operations are the paper's (arXiv cs/0103001):
  * ``forward``: X[k] = (1/N) sum_j x[j] e^{-2 pi i jk/N}      (Eq. E2)
  * ``inverse``: f[j] = sum_k c[k] e^{+2 pi i jk/N}           (Eq. E3, Sec. 3)
  * rank 2: eq5 (1/N, N = rows) and the 2D-IDFT (1/M)
  * ``filter_pipeline``: 2D-IDFT(H .* 2D-DFT(f))              (Sec. 6)
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libb200fft.so")

# fft_status
FFT_OK = 0
STATUS = {0: "FFT_OK", 1: "FFT_E_INVALID_SIZE", 2: "FFT_E_INVALID_ARG", 3: "FFT_E_UNSUPPORTED",
          4: "FFT_E_CUDA", 5: "FFT_E_NCCL", 6: "FFT_E_ALLOC", 7: "FFT_E_STATE"}
# fft_precision
C64, C128 = 0, 1
# fft_filter
FILTER_NONE, FILTER_GAUSS, FILTER_IDEAL_LITERAL, FILTER_IDEAL_LOWPASS = 0, 1, 2, 3
# flags
OUT_TRANSPOSED = 1 << 0
IN_REAL_F32 = 1 << 1
OUT_REAL_F32 = 1 << 2  # NEXT-3 real-to-real Gaussian pipeline (with IN_REAL_F32)

EXPORTS = [
    "fft_plan_create", "fft_plan_create_ex", "fft_plan_set_stream", "fft_plan_workspace_bytes",
    "fft_plan_set_workspace", "fft_forward", "fft_inverse", "fft2d_filter_pipeline", "fft2d_image_filter_u8",
    "fft_forward_paper_tree",
    "fft_execute_host", "fft_nccl_unique_id", "fft_plan_set_comm", "fft_plan_set_host_collectives",
    "fft_plan_set_virtual_ranks",
    "fft_plan_destroy",
    "fft_status_string", "fft_last_error", "fft_plan_last_launch_count", "fft_build_info",
    "fft_plan_set_profiling", "fft_plan_phase_times", "fft_forward_r2c", "fft_inverse_c2r",
]


class FFTError(RuntimeError):
    def __init__(self, status: int, what: str, detail: str):
        super().__init__(f"{what}: {STATUS.get(status, status)}: {detail}")
        self.status = status


_lib = None

# fft_host_allgather_fn / fft_host_barrier_fn (include/b200fft.h)
HOST_ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)
HOST_BARRIER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p)


def load_library(path: str = LIB_PATH) -> ctypes.CDLL:
    """Load libb200fft.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"libb200fft.so not built at {path}; run __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    i64, vp, ci, cd, sz = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
    pp = ctypes.POINTER(vp)
    sig = {
        "fft_plan_create": ([pp, i64, i64, ci], ci),
        "fft_plan_create_ex": ([pp, ctypes.POINTER(i64), ci, i64, ci, ctypes.c_uint], ci),
        "fft_plan_set_stream": ([vp, vp], ci),
        "fft_plan_workspace_bytes": ([vp], sz),
        "fft_plan_set_workspace": ([vp, vp, sz], ci),
        "fft_forward": ([vp, vp, vp], ci),
        "fft_inverse": ([vp, vp, vp], ci),
        "fft2d_filter_pipeline": ([vp, vp, vp, ci, cd], ci),
        "fft_execute_host": ([vp, ci, vp, vp, ci, cd], ci),
        "fft2d_image_filter_u8": ([vp, vp, i64, i64, vp, ci, cd, ci, vp], ci),
        "fft_forward_paper_tree": ([vp, vp, vp], ci),
        "fft_nccl_unique_id": ([ctypes.c_char_p], ci),
        "fft_plan_set_comm": ([vp, ctypes.c_char_p, ci, ci], ci),
        "fft_plan_set_host_collectives": ([vp, ci, ci, HOST_ALLGATHER_FN, HOST_BARRIER_FN, vp], ci),
        "fft_plan_set_virtual_ranks": ([vp, ci], ci),
        "fft_plan_destroy": ([vp], ci),
        "fft_status_string": ([ci], ctypes.c_char_p),
        "fft_last_error": ([], ctypes.c_char_p),
        "fft_plan_last_launch_count": ([vp], ci),
        "fft_build_info": ([], ctypes.c_char_p),
        "fft_plan_set_profiling": ([vp, ci], ci),
        "fft_forward_r2c": ([vp, vp, vp], ci),
        "fft_inverse_c2r": ([vp, vp, vp], ci),
        "fft_plan_phase_times": ([vp, ctypes.POINTER(ctypes.c_float), ci, ctypes.c_char_p, sz], ci),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    _lib = lib
    return lib


def _check(status: int, what: str):
    if status != FFT_OK:
        raise FFTError(status, what, load_library().fft_last_error().decode())


def _ptr(t) -> int:
    """Device (or host) address of a torch tensor / numpy array / int."""
    if t is None:
        return 0
    if isinstance(t, int):
        return t
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    if hasattr(t, "ctypes"):
        return t.ctypes.data
    raise TypeError(f"cannot take the address of {type(t)}")


class Plan:
    """An FFT plan: ``dims`` = (n,) for 1D or (N, M) for 2D; ``batch``
    transforms; precision C64 (complex64) or C128 (complex128)."""

    def __init__(self, dims, batch: int = 1, precision: int = C64, flags: int = 0, stream=None):
        lib = load_library()
        dims = tuple(int(d) for d in (dims if isinstance(dims, (tuple, list)) else (dims,)))
        self.dims, self.batch, self.precision, self.flags = dims, int(batch), precision, flags
        arr = (ctypes.c_int64 * len(dims))(*dims)
        h = ctypes.c_void_p()
        _check(lib.fft_plan_create_ex(ctypes.byref(h), arr, len(dims), self.batch, precision, flags),
               "fft_plan_create_ex")
        self._h = h
        self._keep = []
        if stream is not None:
            self.set_stream(stream)

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream) -> None:
        """``stream``: a torch.cuda.Stream, a raw cudaStream_t int, or None (default)."""
        raw = getattr(stream, "cuda_stream", stream) or 0
        _check(load_library().fft_plan_set_stream(self._h, raw), "fft_plan_set_stream")

    def workspace_bytes(self) -> int:
        return int(load_library().fft_plan_workspace_bytes(self._h))

    def set_workspace(self, tensor) -> None:
        _check(load_library().fft_plan_set_workspace(self._h, _ptr(tensor),
                                                     tensor.numel() * tensor.element_size()),
               "fft_plan_set_workspace")
        self._keep.append(tensor)

    def forward(self, x, out=None):
        out = x if out is None else out
        _check(load_library().fft_forward(self._h, _ptr(x), _ptr(out)), "fft_forward")
        return out

    def inverse(self, x, out=None):
        out = x if out is None else out
        _check(load_library().fft_inverse(self._h, _ptr(x), _ptr(out)), "fft_inverse")
        return out

    def forward_r2c(self, x, out):
        """Real rows / grids -> Hermitian half spectrum (n/2 + 1 bins per row)."""
        _check(load_library().fft_forward_r2c(self._h, _ptr(x), _ptr(out)), "fft_forward_r2c")
        return out

    def inverse_c2r(self, x, out):
        """Hermitian half spectrum -> real rows / grids (unscaled / 1/M)."""
        _check(load_library().fft_inverse_c2r(self._h, _ptr(x), _ptr(out)), "fft_inverse_c2r")
        return out

    def filter_pipeline(self, x, out, filter: int = FILTER_GAUSS, param: float = 0.1):
        _check(load_library().fft2d_filter_pipeline(self._h, _ptr(x), _ptr(out), int(filter),
                                                    float(param)), "fft2d_filter_pipeline")
        return out

    def forward_paper_tree(self, x, out=None):
        """The paper's parallel schedule (Sec. 4): ``x`` = this rank's cyclic
        branch x[q + P j] (virtual ranks: all P branches back to back); rank 0's
        ``out`` receives the whole (1/n) DFT in natural order."""
        _check(load_library().fft_forward_paper_tree(self._h, _ptr(x), _ptr(out)), "fft_forward_paper_tree")
        return out

    def image_filter_u8(self, img, out, filter: int = FILTER_IDEAL_LITERAL, param: float = 340.0,
                        max_val: int = 255, spectrum=None):
        """The paper's image application (Sec. 6): uint8 [batch][h][w] device image ->
        zero-pad to the plan's N x M -> 2D FFT -> x H -> 2D IFFT -> real, round, clamp,
        crop -> uint8 ``out``; optional float32 [batch][N][M] ``spectrum`` |F|."""
        h, w = int(img.shape[-2]), int(img.shape[-1])
        _check(load_library().fft2d_image_filter_u8(self._h, _ptr(img), h, w, _ptr(out), int(filter),
                                                    float(param), int(max_val), _ptr(spectrum)),
               "fft2d_image_filter_u8")
        return out

    def execute_host(self, direction: int, host_in, host_out, filter: int = FILTER_NONE,
                     param: float = 0.0):
        """End to end on host buffers (numpy arrays or CPU tensors, ideally pinned)."""
        _check(load_library().fft_execute_host(self._h, int(direction), _ptr(host_in),
                                               _ptr(host_out), int(filter), float(param)),
               "fft_execute_host")
        return host_out

    def set_comm(self, unique_id: bytes, nranks: int, rank: int) -> None:
        _check(load_library().fft_plan_set_comm(self._h, unique_id, int(nranks), int(rank)),
               "fft_plan_set_comm")

    def set_host_collectives(self, nranks: int, rank: int, allgather, barrier) -> None:
        """Tests on one GPU (fft_plan_set_host_collectives): the fused
        schedules' two collectives by host callables -- ``allgather(mine:
        bytes) -> list of nranks bytes`` (rank order) and ``barrier()`` --
        e.g. over a gloo process group; the data plane is the NCCL path's."""
        def _ag(ctx, mine, out, nbytes):
            try:
                parts = allgather(ctypes.string_at(mine, nbytes))
                blob = b"".join(parts)
                assert len(blob) == nranks * nbytes
                ctypes.memmove(out, blob, len(blob))
                return 0
            except Exception:  # reported to the library as a failed collective
                return 1

        def _bar(ctx):
            try:
                barrier()
                return 0
            except Exception:
                return 1
        self._hc = (HOST_ALLGATHER_FN(_ag), HOST_BARRIER_FN(_bar))  # kept alive with the plan
        _check(load_library().fft_plan_set_host_collectives(self._h, int(nranks), int(rank), self._hc[0],
                                                            self._hc[1], None),
               "fft_plan_set_host_collectives")

    def set_virtual_ranks(self, nranks: int) -> None:
        """Tests: emulate the slab decomposition over ``nranks`` virtual ranks on this GPU."""
        _check(load_library().fft_plan_set_virtual_ranks(self._h, int(nranks)),
               "fft_plan_set_virtual_ranks")

    def set_profiling(self, on: bool = True) -> None:
        """Per-phase CUDA-event timing of later calls (fft_plan_set_profiling)."""
        _check(load_library().fft_plan_set_profiling(self._h, int(bool(on))), "fft_plan_set_profiling")

    def phase_times(self, max_phases: int = 32):
        """[(label, ms), ...] of the last call's phases (waits for it)."""
        ms = (ctypes.c_float * max_phases)()
        buf = ctypes.create_string_buffer(4096)
        n = load_library().fft_plan_phase_times(self._h, ms, max_phases, buf, 4096)
        labels = buf.value.decode().split(";") if n else []
        return [(labels[k] if k < len(labels) else "", float(ms[k])) for k in range(n)]

    def last_launch_count(self) -> int:
        return int(load_library().fft_plan_last_launch_count(self._h))

    def destroy(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            st = load_library().fft_plan_destroy(self._h)
            self._h = ctypes.c_void_p()
            _check(st, "fft_plan_destroy")

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load_library().fft_nccl_unique_id(buf), "fft_nccl_unique_id")
    return buf.raw


def build_info() -> str:
    return load_library().fft_build_info().decode()
