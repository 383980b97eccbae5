// kernels_image.cu -- the paper's own application (Sec. 6, PAPER.md
// P:352-398) as two row kernels around the fused column pass (sm_100a):
//
//   k_image_rows_fwd : an 8-bit image of h x w pixels, zero-padded "on rows
//       and on columns to complete the next power of two" to the
//       plan's N x M grid inside the load (no padded copy is materialised),
//       promoted to complex64, forward row DFT (unnormalised: eq5's
//       "FFT on rows -> x M").
//   [k_cols / k_cols_pipe MODE 2 : column DFT -> |F| spectrum (optional,
//       P:369-373) -> x H(u,v) (Eq. filtro, or the Gaussian) /
//       (N M) -> column inverse DFT]
//   k_image_rows_inv : inverse row DFT (2D-IDFT) with the image
//       epilogue fused into the store: real part, round half up, clamp to
//       [0, max_val], crop to h x w, store 8-bit (the "image filtered" of
//       P:394, its digital-image range f(x,y) in Z+ u {0}).
//
// Both row kernels are the engine of fft_engine.cuh with different load /
// store epilogues; every arithmetic step runs here, none on the host.
#include <cstdint>

#include "fft_engine.cuh"
#include "launch.h"

namespace b200fft {

namespace {

template <int R, int E, int W>
__global__ void __launch_bounds__(W*(R / E)) k_image_rows_fwd(const uint8_t* __restrict__ in, float2* __restrict__ out,
                                                              int64_t nrows, int64_t N, int64_t h, int64_t w,
                                                              const float2* __restrict__ tw) {
    using F = LineFFT<float, R, E, false>;
    B200FFT_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* smem = reinterpret_cast<float2*>(smem_raw);
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int64_t row = (int64_t)blockIdx.x * W + t;
    const bool valid = row < nrows;
    const int64_t img = row / N, x = row - img * N;
    float2 v[E];
    if (valid && x < h) {
        const uint8_t* src = in + (img * h + x) * w;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int64_t c = lt + F::TPL * m;
            v[F::pos_in(m)] = mk(c < w ? (float)__ldg(src + c) : 0.0f, 0.0f);
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = mk(0.0f, 0.0f);
    }
    F::run(v, smem + t * F::LS, lt, tw);
    if (valid) {
        float2* o = out + row * R + lt;
#pragma unroll
        for (int m = 0; m < E; ++m) o[F::TPL * m] = v[F::pos_out(m)];
    }
}

template <int R, int E, int W>
__global__ void __launch_bounds__(W*(R / E)) k_image_rows_inv(const float2* __restrict__ in, uint8_t* __restrict__ out,
                                                              int64_t nrows, int64_t N, int64_t h, int64_t w,
                                                              float max_val, const float2* __restrict__ tw) {
    using F = LineFFT<float, R, E, true>;
    B200FFT_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    float2* smem = reinterpret_cast<float2*>(smem_raw);
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int64_t row = (int64_t)blockIdx.x * W + t;
    const int64_t img = row / N, x = row - img * N;
    // rows x >= h are cropped away; their lines still join the CTA's barriers
    const bool keep = row < nrows && x < h;
    float2 v[E];
    if (keep) {
        const float2* src = in + row * R + lt;
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = src[F::TPL * m];
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = mk(0.0f, 0.0f);
    }
    F::run(v, smem + t * F::LS, lt, tw);
    if (keep) {
        uint8_t* o = out + (img * h + x) * w;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int64_t c = lt + F::TPL * m;
            if (c < w) {
                const float q = fminf(fmaxf(floorf(v[F::pos_out(m)].x + 0.5f), 0.0f), max_val);
                o[c] = (uint8_t)q;
            }
        }
    }
}

template <int R>
constexpr int img_e() { return R < 16 ? R : 16; }
template <int R>
constexpr int img_w() { return (R / img_e<R>()) >= 256 ? 1 : 256 / (R / img_e<R>()); }

template <int R>
cudaError_t image_rows_t(bool inv, const void* in, void* out, int64_t nrows, int64_t N, int64_t h, int64_t w,
                         int max_val, const void* tw, cudaStream_t st) {
    constexpr int E = img_e<R>(), W = img_w<R>(), TPL = R / E;
    using F = LineFFT<float, R, E, false>;
    constexpr size_t smem = sizeof(float2) * W * F::LS;
    {
        cudaError_t e = kernel_setup((const void*)k_image_rows_fwd<R, E, W>, 0, smem, nullptr);
        if (e == cudaSuccess) e = kernel_setup((const void*)k_image_rows_inv<R, E, W>, 0, smem, nullptr);
        if (e != cudaSuccess) return e;
    }
    if (nrows <= 0) return cudaSuccess;
    const unsigned grid = (unsigned)((nrows + W - 1) / W);
    const float2* t = reinterpret_cast<const float2*>(tw) + tw_base(R);
    if (!inv)
        return launch_pdl(k_image_rows_fwd<R, E, W>, dim3(grid), dim3(W * TPL), smem, st,
                          reinterpret_cast<const uint8_t*>(in), reinterpret_cast<float2*>(out), nrows, N, h, w, t);
    return launch_pdl(k_image_rows_inv<R, E, W>, dim3(grid), dim3(W * TPL), smem, st,
                      reinterpret_cast<const float2*>(in), reinterpret_cast<uint8_t*>(out), nrows, N, h, w,
                      (float)max_val, t);
}

}  // namespace

cudaError_t launch_image_rows(bool inv, int64_t M, const void* in, void* out, int64_t nrows, int64_t N, int64_t h,
                              int64_t w, int max_val, const void* tw, cudaStream_t st) {
    switch (M) {
#define B200_IMG_CASE(r) \
    case r: return image_rows_t<r>(inv, in, out, nrows, N, h, w, max_val, tw, st);
        B200_IMG_CASE(1) B200_IMG_CASE(2) B200_IMG_CASE(4) B200_IMG_CASE(8) B200_IMG_CASE(16)
        B200_IMG_CASE(32) B200_IMG_CASE(64) B200_IMG_CASE(128) B200_IMG_CASE(256)
        B200_IMG_CASE(512) B200_IMG_CASE(1024) B200_IMG_CASE(2048) B200_IMG_CASE(4096)
        B200_IMG_CASE(8192)
#undef B200_IMG_CASE
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace b200fft
