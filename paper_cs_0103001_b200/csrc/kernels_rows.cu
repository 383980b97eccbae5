// kernels_rows.cu -- instantiations and launcher of kernel family A (rows).
#include "fft_engine.cuh"
#include "launch.h"

namespace b200fft {

namespace {

template <typename T, int R, bool INV, bool REAL_IN>
cudaError_t rows_t(const void* in, void* out, int64_t batch, double scale, const void* tw, int in_sh, int out_sh,
                   cudaStream_t st) {
    constexpr int E = R < 16 ? R : 16;
    constexpr int TPL = R / E;
    constexpr int W = TPL >= 256 ? 1 : 256 / TPL;
    using F = LineFFT<T, R, E, INV>;
    constexpr size_t smem = sizeof(cpx<T>) * W * F::LS;
    auto kern = k_rows<T, R, E, W, INV, REAL_IN>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t grid = (batch + W - 1) / W;
    kern<<<(unsigned)grid, W * TPL, smem, st>>>(in, reinterpret_cast<cpx<T>*>(out), batch, (T)scale,
                                                 reinterpret_cast<const cpx<T>*>(tw) + tw_base(R), in_sh, out_sh);
    return cudaGetLastError();
}

template <typename T, bool INV, bool REAL_IN>
cudaError_t rows_r(int64_t R, const void* in, void* out, int64_t batch, double scale, const void* tw, int in_sh,
                   int out_sh, cudaStream_t st) {
    switch (R) {
#define B200_ROWS_CASE(r) \
    case r: return rows_t<T, r, INV, REAL_IN>(in, out, batch, scale, tw, in_sh, out_sh, st);
        B200_ROWS_CASE(1) B200_ROWS_CASE(2) B200_ROWS_CASE(4) B200_ROWS_CASE(8) B200_ROWS_CASE(16)
        B200_ROWS_CASE(32) B200_ROWS_CASE(64) B200_ROWS_CASE(128) B200_ROWS_CASE(256)
        B200_ROWS_CASE(512) B200_ROWS_CASE(1024) B200_ROWS_CASE(2048) B200_ROWS_CASE(4096)
        B200_ROWS_CASE(8192)
#undef B200_ROWS_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_rows(int prec, bool inv, bool real_in, int64_t R, const void* in, void* out,
                        int64_t batch, double scale, const void* tw, cudaStream_t st, int in_sh, int out_sh) {
    if (prec == 0) {
        if (real_in) return rows_r<float, false, true>(R, in, out, batch, scale, tw, in_sh, out_sh, st);
        return inv ? rows_r<float, true, false>(R, in, out, batch, scale, tw, in_sh, out_sh, st)
                   : rows_r<float, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, st);
    }
    if (real_in) return cudaErrorInvalidValue;
    return inv ? rows_r<double, true, false>(R, in, out, batch, scale, tw, in_sh, out_sh, st)
               : rows_r<double, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, st);
}

}  // namespace b200fft
