// kernels_real.cu -- instantiations and launchers of the real-input /
// real-output row kernels (fft_real.cuh).
#include "fft_real.cuh"
#include "launch.h"

namespace b200fft {

namespace {

// R = M / 2 complex points per row; E values per thread, W rows per CTA
template <typename T, int R, bool C2R>
cudaError_t real_rows_t(const void* in, void* out, int64_t batch, double scale, const void* tw, const void* rtw,
                        cudaStream_t st, int64_t ld) {
    if (ld <= 0) ld = R + 1;
    constexpr int E = R < 16 ? R : 16;
    constexpr int TPL = R / E;
    constexpr int W = TPL >= 256 ? 1 : 256 / TPL;
    using F = LineFFT<T, R, E, C2R>;
    constexpr size_t smem = sizeof(cpx<T>) * W * F::LS;
    const void* kern = C2R ? (const void*)k_rows_c2r<T, R, E, W> : (const void*)k_rows_r2c<T, R, E, W>;
    cudaError_t e = kernel_setup(kern, 0, smem, nullptr);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    const dim3 grid((unsigned)((batch + W - 1) / W));
    const cpx<T>* a_tw = reinterpret_cast<const cpx<T>*>(tw) + tw_base(R);
    const cpx<T>* a_rtw = reinterpret_cast<const cpx<T>*>(rtw);
    if constexpr (C2R)
        return launch_pdl(k_rows_c2r<T, R, E, W>, grid, dim3(W * TPL), smem, st,
                          reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<T*>(out), batch, (T)scale, a_tw,
                          a_rtw, ld);
    else
        return launch_pdl(k_rows_r2c<T, R, E, W>, grid, dim3(W * TPL), smem, st, reinterpret_cast<const T*>(in),
                          reinterpret_cast<cpx<T>*>(out), batch, (T)scale, a_tw, a_rtw, ld);
}

template <typename T, bool C2R>
cudaError_t real_rows_r(int64_t M, const void* in, void* out, int64_t batch, double scale, const void* tw,
                        const void* rtw, cudaStream_t st, int64_t ld) {
    switch (M / 2) {
#define B200_REAL_CASE(r) \
    case r: return real_rows_t<T, r, C2R>(in, out, batch, scale, tw, rtw, st, ld);
        B200_REAL_CASE(1) B200_REAL_CASE(2) B200_REAL_CASE(4) B200_REAL_CASE(8) B200_REAL_CASE(16)
        B200_REAL_CASE(32) B200_REAL_CASE(64) B200_REAL_CASE(128) B200_REAL_CASE(256) B200_REAL_CASE(512)
        B200_REAL_CASE(1024) B200_REAL_CASE(2048) B200_REAL_CASE(4096)
#undef B200_REAL_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_rows_r2c(int prec, int64_t M, const void* in, void* out, int64_t batch, double scale,
                            const void* tw, const void* rtw, cudaStream_t st, int64_t ld) {
    return prec == 0 ? real_rows_r<float, false>(M, in, out, batch, scale, tw, rtw, st, ld)
                     : real_rows_r<double, false>(M, in, out, batch, scale, tw, rtw, st, ld);
}

cudaError_t launch_rows_c2r(int prec, int64_t M, const void* in, void* out, int64_t batch, double scale,
                            const void* tw, const void* rtw, cudaStream_t st, int64_t ld) {
    return prec == 0 ? real_rows_r<float, true>(M, in, out, batch, scale, tw, rtw, st, ld)
                     : real_rows_r<double, true>(M, in, out, batch, scale, tw, rtw, st, ld);
}

}  // namespace b200fft
