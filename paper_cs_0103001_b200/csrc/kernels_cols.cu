// kernels_cols.cu -- instantiations and launcher of kernel family B (columns,
// and the fused column forward -> filter -> column inverse of the pipeline).
#include "fft_cols_pipe.cuh"
#include "fft_engine.cuh"
#include "launch.h"

#include <cstdlib>

namespace b200fft {

namespace {

// persistent double-buffered variant (fft_cols_pipe.cuh), complex64,
// 256 <= R <= 4096: W columns per tile so that two tiles fit in smem
template <int R> constexpr int pipe_w() {
    return R >= 4096 ? 2 : (R >= 2048 ? 4 : (R >= 1024 ? 8 : (R >= 256 ? 16 : (R >= 128 ? 32 : 64))));
}

template <int R, int MODE, int WF = 0, int NS = 2>
cudaError_t cols_pipe_t(const void* in, void* out, int64_t S, int64_t nimg, double scale, const void* tw,
                        const FilterArgs& f, cudaStream_t st) {
    constexpr int E = 16, W = WF ? WF : pipe_w<R>();
    using G = ColsPipeCfg<float, R, W, NS>;
    auto kern = k_cols_pipe<float, R, E, W, MODE, NS>;
    int grid_max = 0;
    {
        cudaError_t e = kernel_setup((const void*)kern, W * (R / E), G::SMEM_BYTES, &grid_max);
        if (e != cudaSuccess) return e;
    }
    if (S <= 0 || nimg <= 0) return cudaSuccess;
    const int64_t tiles = (S + W - 1) / W * nimg;
    const int grid = (int)(tiles < grid_max ? tiles : grid_max);
    return launch_pdl(kern, dim3(grid), dim3(W * (R / E)), G::SMEM_BYTES, st, reinterpret_cast<const float2*>(in),
                      reinterpret_cast<float2*>(out), S, nimg, (float)scale,
                      reinterpret_cast<const float2*>(tw) + tw_base(R), f);
}

template <int MODE>
cudaError_t cols_pipe_r(int64_t R, const void* in, void* out, int64_t S, int64_t nimg, double scale, const void* tw,
                        const FilterArgs& f, cudaStream_t st) {
    switch (R) {
        case 64: return cols_pipe_t<64, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 128: return cols_pipe_t<128, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 256: return cols_pipe_t<256, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 512: return cols_pipe_t<512, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 1024: return cols_pipe_t<1024, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 2048: return cols_pipe_t<2048, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 4096: return cols_pipe_t<4096, MODE>(in, out, S, nimg, scale, tw, f, st);
        default: return cudaErrorInvalidValue;
    }
}

bool use_cols_pipe(int prec, int64_t R) {
    static const bool off = [] {
        const char* e = getenv("B200FFT_NO_COLPIPE");
        return e && e[0] == '1';
    }();
    return !off && prec == 0 && R >= 256 && R <= 4096;
}

template <typename T> constexpr int cols_budget() { return sizeof(T) == 4 ? 16384 : 8192; }

template <typename T, int R> constexpr int cols_e() { return R < 32 ? (R < 16 ? R : 16) : 32; }
template <typename T, int R> constexpr int cols_w() {
    return cols_budget<T>() / R > 16 ? 16 : (cols_budget<T>() / R < 2 ? 2 : cols_budget<T>() / R);
}

template <typename T, int R, int MODE, int W = cols_w<T, R>(), int E = cols_e<T, R>(), int MINB = 0>
cudaError_t cols_t(const void* in, void* out, int64_t S, int64_t nimg, double scale, const void* tw,
                   const FilterArgs& f, cudaStream_t st) {
    constexpr int TPL = R / E;
    using F = LineFFT<T, R, E, MODE == 1>;
    constexpr size_t smem = sizeof(cpx<T>) * W * cols_ls<T, R, W>();
    static_assert(smem <= 227 * 1024, "column tile exceeds shared memory");
    auto kern = k_cols<T, R, E, W, MODE, MINB>;
    {
        cudaError_t e = kernel_setup((const void*)kern, 0, smem, nullptr);
        if (e != cudaSuccess) return e;
    }
    if (S <= 0 || nimg <= 0) return cudaSuccess;
    dim3 grid((unsigned)((S + W - 1) / W), (unsigned)nimg);
    return launch_pdl(kern, grid, dim3(W * TPL), smem, st, reinterpret_cast<const cpx<T>*>(in),
                      reinterpret_cast<cpx<T>*>(out), S, (T)scale, reinterpret_cast<const cpx<T>*>(tw) + tw_base(R), f);
}

template <typename T, int MODE>
cudaError_t cols_r(int64_t R, const void* in, void* out, int64_t S, int64_t nimg, double scale,
                   const void* tw, const FilterArgs& f, cudaStream_t st) {
    switch (R) {
#define B200_COLS_CASE(r) \
    case r: return cols_t<T, r, MODE>(in, out, S, nimg, scale, tw, f, st);
        B200_COLS_CASE(1) B200_COLS_CASE(2) B200_COLS_CASE(4) B200_COLS_CASE(8) B200_COLS_CASE(16)
        B200_COLS_CASE(32) B200_COLS_CASE(64) B200_COLS_CASE(128) B200_COLS_CASE(256)
        B200_COLS_CASE(512) B200_COLS_CASE(1024) B200_COLS_CASE(4096)
#undef B200_COLS_CASE
        case 2048: return cols_t<T, 2048, MODE>(in, out, S, nimg, scale, tw, f, st);
        case 8192:
            if constexpr (sizeof(T) == 4) return cols_t<T, 8192, MODE>(in, out, S, nimg, scale, tw, f, st);
            return cudaErrorInvalidValue;
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

// four-step column passes (N = 4096 columns, and column slabs whose width is
// not a power of two): per-CTA k_cols tiles of 16 columns, E = 16; the
// 128-point fwd * g * inv pass capped at 56 registers (9 CTAs/SM) -- the
// measured best of the tile / ring / register configurations (profiles/README.md)
template <int MODE>
cudaError_t cols4_r(int64_t R, const void* in, void* out, int64_t S, int64_t nimg, double scale, const void* tw,
                    const FilterArgs& f, cudaStream_t st) {
    if (R == 64) return cols_t<float, 64, MODE, 16, 16>(in, out, S, nimg, scale, tw, f, st);
    if (R == 128) return cols_t<float, 128, MODE, 16, 16, 9>(in, out, S, nimg, scale, tw, f, st);
    return cols_pipe_r<MODE>(R, in, out, S, nimg, scale, tw, f, st);
}

cudaError_t launch_cols_fourstep(int mode, int64_t R, const void* in, void* out, int64_t S, int64_t nimg,
                                 double scale, const void* tw, const FilterArgs& f, cudaStream_t st) {
    if (R < 64 || R > 4096) return cudaErrorInvalidValue;
    switch (mode) {
        case 2: return cols4_r<2>(R, in, out, S, nimg, scale, tw, f, st);
        case 3: return cols4_r<3>(R, in, out, S, nimg, scale, tw, f, st);
        case 4: return cols4_r<4>(R, in, out, S, nimg, scale, tw, f, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_cols(int prec, int mode, int64_t R, const void* in, void* out, int64_t S,
                        int64_t nimg, double scale, const void* tw, const FilterArgs& f,
                        cudaStream_t st) {
    if (use_cols_pipe(prec, R)) {
        switch (mode) {
            case 0: return cols_pipe_r<0>(R, in, out, S, nimg, scale, tw, f, st);
            case 1: return cols_pipe_r<1>(R, in, out, S, nimg, scale, tw, f, st);
            case 2: return cols_pipe_r<2>(R, in, out, S, nimg, scale, tw, f, st);
        }
    }
    if (prec == 0) {
        switch (mode) {
            case 0: return cols_r<float, 0>(R, in, out, S, nimg, scale, tw, f, st);
            case 1: return cols_r<float, 1>(R, in, out, S, nimg, scale, tw, f, st);
            case 2: return cols_r<float, 2>(R, in, out, S, nimg, scale, tw, f, st);
        }
    } else {
        switch (mode) {
            case 0: return cols_r<double, 0>(R, in, out, S, nimg, scale, tw, f, st);
            case 1: return cols_r<double, 1>(R, in, out, S, nimg, scale, tw, f, st);
            case 2: return cols_r<double, 2>(R, in, out, S, nimg, scale, tw, f, st);
        }
    }
    return cudaErrorInvalidValue;
}

}  // namespace b200fft
