// kernels_pass.cu -- instantiations and launcher of kernel family C (one
// global Stockham pass of a multi-pass transform, L > 8192).
#include "fft_engine.cuh"
#include "launch.h"

namespace b200fft {

namespace {

template <typename T, int R, bool INV, int WF = 0>
cudaError_t pass_t(const void* in, void* out, int64_t L, int64_t Ns, int64_t batch, double scale,
                   const void* tw, const void* pa, const void* pb, int klo_sh, cudaStream_t st) {
    constexpr int E = 16;
    constexpr int TPL = R / E;
    constexpr int W = WF ? WF : ((R >= 1024) ? 8 : 16);
    using F = LineFFT<T, R, E, INV>;
    constexpr size_t smem = sizeof(cpx<T>) * W * F::LS;
    auto kern = k_pass<T, R, E, W, INV>;
    {
        cudaError_t e = kernel_setup((const void*)kern, 0, smem, nullptr);
        if (e != cudaSuccess) return e;
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t LR = L / R;
    if (LR % W != 0 || (Ns > 1 && Ns < W)) return cudaErrorInvalidValue;
    const int64_t nlines = batch * LR;
    const int64_t grid = nlines / W;
    kern<<<(unsigned)grid, W * TPL, smem, st>>>(
        reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out), L, Ns, nlines, (T)scale,
        reinterpret_cast<const cpx<T>*>(tw) + tw_base(R), reinterpret_cast<const cpx<T>*>(pa),
        reinterpret_cast<const cpx<T>*>(pb), klo_sh);
    return cudaGetLastError();
}

template <typename T, bool INV>
cudaError_t pass_r(int64_t R, const void* in, void* out, int64_t L, int64_t Ns, int64_t batch,
                   double scale, const void* tw, const void* pa, const void* pb, int klo_sh,
                   cudaStream_t st) {
    switch (R) {
        case 128: return pass_t<T, 128, INV>(in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
        case 256: return pass_t<T, 256, INV>(in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
        case 512: return pass_t<T, 512, INV>(in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
        case 1024: return pass_t<T, 1024, INV>(in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

cudaError_t launch_pass(int prec, bool inv, int64_t R, const void* in, void* out, int64_t L,
                        int64_t Ns, int64_t batch, double scale, const void* tw, const void* pa,
                        const void* pb, int klo_sh, cudaStream_t st) {
    if (prec == 0)
        return inv ? pass_r<float, true>(R, in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st)
                   : pass_r<float, false>(R, in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
    return inv ? pass_r<double, true>(R, in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st)
               : pass_r<double, false>(R, in, out, L, Ns, batch, scale, tw, pa, pb, klo_sh, st);
}

}  // namespace b200fft
