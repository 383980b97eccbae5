// kernels_rows.cu -- instantiations and launcher of kernel family A (rows):
// the per-CTA k_rows (any R, any precision, blocked layouts) and the
// persistent TMA-fed k_rows_tma (complex64, 256 <= R <= 8192, natural rows).
#include <cstdlib>

#include "fft_engine.cuh"
#include "fft_tma.cuh"
#include "launch.h"

namespace b200fft {

bool pdl_enabled() {
    static const bool on = [] {
        const char* v = getenv("B200FFT_PDL");
        return !(v && v[0] == '0');
    }();
    return on;
}

bool& pdl_hint() {
    static thread_local bool hint = false;
    return hint;
}

namespace {

template <typename T, int R, bool INV, bool REAL_IN, bool FILT>
cudaError_t rows_t(const void* in, void* out, int64_t batch, double scale, const void* tw, int in_sh, int out_sh,
                   const void* rowfilt, cudaStream_t st, const BlockPtrs* ibp, const BlockPtrs* obp) {
    constexpr int E = R < 16 ? R : 16;
    constexpr int TPL = R / E;
    constexpr int W = TPL >= 256 ? 1 : 256 / TPL;
    using F = LineFFT<T, R, E, INV>;
    constexpr size_t smem = sizeof(cpx<T>) * W * F::LS;
    auto kern = k_rows<T, R, E, W, INV, REAL_IN, FILT>;
    {
        cudaError_t e = kernel_setup((const void*)kern, 0, smem, nullptr);
        if (e != cudaSuccess) return e;
    }
    if (batch <= 0) return cudaSuccess;
    // blocked layouts: the given block pointers, or local blocks of batch
    // rows x 2^sh elements one after the other
    BlockPtrs ib{}, ob{};
    auto blocks = [&](int sh, const void* base, const BlockPtrs* given, size_t eb, BlockPtrs& b) {
        if (sh < 0) return true;
        if ((R >> sh) > kMaxBlocks || (R >> sh) < 1) return false;
        if (given) {
            b = *given;
        } else {
            for (int q = 0; q < (R >> sh); ++q)
                b.p[q] = const_cast<char*>(reinterpret_cast<const char*>(base)) + (size_t)q * ((size_t)batch << sh) * eb;
        }
        return true;
    };
    if (!blocks(in_sh, in, ibp, REAL_IN ? sizeof(float) : sizeof(cpx<T>), ib) ||
        !blocks(out_sh, out, obp, sizeof(cpx<T>), ob))
        return cudaErrorInvalidValue;
    const int64_t grid = (batch + W - 1) / W;
    return launch_pdl(kern, dim3((unsigned)grid), dim3(W * TPL), smem, st, in, reinterpret_cast<cpx<T>*>(out), batch,
                      (T)scale, reinterpret_cast<const cpx<T>*>(tw) + tw_base(R), in_sh, out_sh,
                      reinterpret_cast<const T*>(rowfilt), ib, ob);
}

template <typename T, bool INV, bool REAL_IN, bool FILT>
cudaError_t rows_r(int64_t R, const void* in, void* out, int64_t batch, double scale, const void* tw, int in_sh,
                   int out_sh, const void* rowfilt, cudaStream_t st, const BlockPtrs* ib, const BlockPtrs* ob) {
    switch (R) {
#define B200_ROWS_CASE(r) \
    case r: return rows_t<T, r, INV, REAL_IN, FILT>(in, out, batch, scale, tw, in_sh, out_sh, rowfilt, st, ib, ob);
        B200_ROWS_CASE(1) B200_ROWS_CASE(2) B200_ROWS_CASE(4) B200_ROWS_CASE(8) B200_ROWS_CASE(16)
        B200_ROWS_CASE(32) B200_ROWS_CASE(64) B200_ROWS_CASE(128) B200_ROWS_CASE(256)
        B200_ROWS_CASE(512) B200_ROWS_CASE(1024) B200_ROWS_CASE(2048) B200_ROWS_CASE(4096)
        B200_ROWS_CASE(8192)
#undef B200_ROWS_CASE
        default: return cudaErrorInvalidValue;
    }
}

// persistent TMA-fed variant (fft_tma.cuh): 3 stages of ~64 KiB, 512 threads
template <typename T, int R, bool INV, bool REAL_IN, bool FILT, bool TRANS = false, int PAIR = 0, int E = 16,
          int OCC = 1, int STAGE_KB = 64>
cudaError_t rows_tma_t(const void* in, void* out, int64_t batch, double scale, const void* tw, const void* rowfilt,
                       cudaStream_t st, bool pdl = false) {
    constexpr int W = (int)((STAGE_KB * 1024) / (R * sizeof(cpx<T>))) < 1
                          ? 1
                          : (int)((STAGE_KB * 1024) / (R * sizeof(cpx<T>)));
    // OCC CTAs per SM (registers capped): one stage each, or (OCC = 3, the
    // C2 lesson) two smaller stages each
    constexpr int STAGES = OCC == 3 ? 2 : (OCC > 1 && STAGE_KB >= 64 ? 1 : 3);
    using G = RowsTmaCfg<T, R, W, REAL_IN, STAGES>;
    auto kern = k_rows_tma<T, R, E, W, INV, REAL_IN, STAGES, FILT, TRANS, PAIR, OCC>;
    int grid_max = 0;
    {
        cudaError_t e = kernel_setup((const void*)kern, W * (R / E), G::SMEM_BYTES, &grid_max);
        if (e != cudaSuccess) return e;
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t tiles = (batch + W - 1) / W;
    const int grid = (int)(tiles < grid_max ? tiles : grid_max);
    cpx<T>* a_out = reinterpret_cast<cpx<T>*>(out);
    const cpx<T>* a_tw = reinterpret_cast<const cpx<T>*>(tw) + tw_base(R, ml_of(E));
    const T* a_filt = reinterpret_cast<const T*>(rowfilt);
    // timing experiments (wrong results): B200FFT_ROWS_XO with B200FFT_ALLOW_WRONG=1;
    // 1 = no FFT arithmetic / exchanges, 2 = no stores
    static const int xo = [] {
        const char* w = getenv("B200FFT_ALLOW_WRONG");
        const char* v = getenv("B200FFT_ROWS_XO");
        return (w && w[0] == '1' && v) ? atoi(v) : 0;
    }();
    if (pdl && pdl_enabled()) {  // may start on the SMs the previous kernel's CTAs leave (it waits for its results)
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.gridDim = dim3((unsigned)grid);
        cfg.blockDim = dim3(W * (R / E));
        cfg.dynamicSmemBytes = G::SMEM_BYTES;
        cfg.stream = st;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        return cudaLaunchKernelEx(&cfg, kern, in, a_out, batch, (T)scale, a_tw, a_filt, xo);
    }
    kern<<<grid, W * (R / E), G::SMEM_BYTES, st>>>(in, a_out, batch, (T)scale, a_tw, a_filt, xo);
    return cudaGetLastError();
}

// 8192-point complex64 rows: two independent 256-thread groups, E = 32,
// radix-32 steps (fft_tma.cuh k_rows_tma_g); B200FFT_ROWS_G2=0 selects the
// one-group radix-16 k_rows_tma (the earlier form)
template <bool INV, bool FILT>
cudaError_t rows_g2_8192(const void* in, void* out, int64_t batch, double scale, const void* tw, const void* rowfilt,
                         cudaStream_t st) {
    constexpr int R = 8192, E = 32, NG = 2, STAGES = 3, ML = 5;
    using G = RowsTmaCfg<float, R, 1, false, STAGES>;
    auto kern = k_rows_tma_g<float, R, E, NG, INV, STAGES, FILT, ML>;
    int grid_max = 0;
    cudaError_t e = kernel_setup((const void*)kern, NG * (R / E), G::SMEM_BYTES, &grid_max);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    const int grid = (int)(batch < grid_max ? batch : grid_max);
    kern<<<grid, NG * (R / E), G::SMEM_BYTES, st>>>(in, reinterpret_cast<float2*>(out), batch, (float)scale,
                                                     reinterpret_cast<const float2*>(tw) + tw_base(R, ML),
                                                     reinterpret_cast<const float*>(rowfilt));
    return cudaGetLastError();
}

bool rows_g2() {
    const char* v = getenv("B200FFT_ROWS_G2");
    return !(v && v[0] == '0');
}

template <bool INV, bool REAL_IN, bool FILT>
cudaError_t rows_tma_r(int64_t R, const void* in, void* out, int64_t batch, double scale, const void* tw,
                       const void* rowfilt, cudaStream_t st) {
    if constexpr (!REAL_IN) {
        if (R == 8192 && rows_g2()) return rows_g2_8192<INV, FILT>(in, out, batch, scale, tw, rowfilt, st);
    }
    switch (R) {
        case 256: return rows_tma_t<float, 256, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        case 512: return rows_tma_t<float, 512, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        case 1024: return rows_tma_t<float, 1024, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        case 2048: return rows_tma_t<float, 2048, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        case 4096: return rows_tma_t<float, 4096, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        case 8192: return rows_tma_t<float, 8192, INV, REAL_IN, FILT>(in, out, batch, scale, tw, rowfilt, st);
        default: return cudaErrorInvalidValue;
    }
}

bool use_tma_rows(int prec, int64_t R, int in_sh, int out_sh) {
    static const bool off = [] {
        const char* e = getenv("B200FFT_NO_TMA");
        return e && e[0] == '1';
    }();
    return !off && prec == 0 && R >= 256 && R <= 8192 && in_sh < 0 && out_sh < 0;
}

template <bool REAL_IN, int PAIR = 0>
cudaError_t rows_filter_trans_r(int64_t R, const void* in, void* out, int64_t batch, double scale, const void* tw,
                                const void* rowfilt, cudaStream_t st, bool pdl) {
    switch (R) {
        case 256:
            return rows_tma_t<float, 256, false, REAL_IN, true, true, PAIR>(in, out, batch, scale, tw, rowfilt, st, pdl);
        case 512:
            return rows_tma_t<float, 512, false, REAL_IN, true, true, PAIR>(in, out, batch, scale, tw, rowfilt, st, pdl);
        case 1024:
            return rows_tma_t<float, 1024, false, REAL_IN, true, true, PAIR>(in, out, batch, scale, tw, rowfilt, st, pdl);
        case 2048:
            return rows_tma_t<float, 2048, false, REAL_IN, true, true, PAIR>(in, out, batch, scale, tw, rowfilt, st, pdl);
        default: return cudaErrorInvalidValue;
    }
}


// both passes of the square real-pair pipeline in one cooperative launch
// (fft_tma.cuh k_rows_tma2); 3 stages of ~64 KiB, 512 threads, one CTA per SM
// E = 16, tiles of ~64 KiB (4 line pairs at R = 2048), 3 stages.  (8-pair
// tiles with E = 32 and one 128 KiB stage -- one tile per CTA and pass --
// measured 37.9-38.9 us with radix-16 steps, 43.0 with radix-32 (spills):
// profiles/README.md)
template <int R, int PAIR2>
cudaError_t rows2_t(const void* in, void* mid, void* out, double scale1, const void* filt1, double scale2,
                    const void* filt2, const void* tw, unsigned long long* gbar, cudaStream_t st) {
    constexpr int E = 16, STAGES = 3, MLX = 0;
    constexpr int W = (int)((64 * 1024) / (R * sizeof(float2)));
    using G = RowsTmaCfg<float, R, W, false, STAGES>;
    auto kern = k_rows_tma2<R, E, W, STAGES, PAIR2, MLX>;
    const size_t smem = G::SMEM_BYTES + 8 * STAGES;  // a second set of stage barriers
    int grid_max = 0;
    cudaError_t e = kernel_setup((const void*)kern, W * (R / E), smem, &grid_max);
    if (e != cudaSuccess) return e;
    const int64_t lines = R / 2;  // row pairs per pass
    const int64_t tiles = (lines + W - 1) / W;
    const int grid = (int)(tiles < grid_max ? tiles : grid_max);
    static const int xo = [] {
        const char* w = getenv("B200FFT_ALLOW_WRONG");
        const char* v = getenv("B200FFT_ROWS_XO");
        return (w && w[0] == '1' && v) ? atoi(v) : 0;
    }();
    const void* a_in = in;
    float2* a_mid = reinterpret_cast<float2*>(mid);
    void* a_out = out;
    int64_t a_lines = lines;
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(R, MLX ? MLX : ml_of(E));
    float a_s1 = (float)scale1, a_s2 = (float)scale2;
    const float* a_f1 = reinterpret_cast<const float*>(filt1);
    const float* a_f2 = reinterpret_cast<const float*>(filt2);
    int a_xo = xo;
    void* args[] = {&a_in, &a_mid, &a_out, &a_lines, &a_tw, &a_s1, &a_f1, &a_s2, &a_f2, &gbar, &a_xo};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(W * (R / E));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, (const void*)kern, args);
}

}  // namespace

bool rows_filter2_supported(int prec, int64_t N, int64_t M) {
    const char* e = getenv("B200FFT_PIPE_FUSED2");  // "0": the two-launch form (read per call: tests cover both)
    return !(e && e[0] == '0') && N == M && rows_filter_transposed_supported(prec, N) && N >= 512;
}

cudaError_t launch_rows_filter2(int64_t R, const void* in, void* mid, void* out, double scale1, const void* filt1,
                                double scale2, const void* filt2, const void* tw, int pair2, unsigned long long* gbar,
                                cudaStream_t st) {
    if (pair2 != 2) return cudaErrorInvalidValue;  // complex output only (the C3 form)
    switch (R) {
#define B200_R2_CASE(r) \
    case r: return rows2_t<r, 2>(in, mid, out, scale1, filt1, scale2, filt2, tw, gbar, st);
        B200_R2_CASE(512) B200_R2_CASE(1024) B200_R2_CASE(2048)
#undef B200_R2_CASE
        default: return cudaErrorInvalidValue;
    }
}

namespace {
}  // namespace

bool rows_filter_transposed_supported(int prec, int64_t R) {
    return use_tma_rows(prec, R, -1, -1) && R <= 2048;
}

cudaError_t launch_rows_filter_transposed(bool real_in, int64_t R, const void* in, void* out, int64_t batch,
                                          double scale, const void* tw, const void* rowfilt, cudaStream_t st,
                                          int pair, bool pdl) {
    if (pair == 2) return rows_filter_trans_r<false, 2>(R, in, out, batch, scale, tw, rowfilt, st, pdl);
    if (pair) return rows_filter_trans_r<false, 1>(R, in, out, batch, scale, tw, rowfilt, st, pdl);
    return real_in ? rows_filter_trans_r<true>(R, in, out, batch, scale, tw, rowfilt, st, pdl)
                   : rows_filter_trans_r<false>(R, in, out, batch, scale, tw, rowfilt, st, pdl);
}

cudaError_t launch_rows(int prec, bool inv, bool real_in, int64_t R, const void* in, void* out,
                        int64_t batch, double scale, const void* tw, cudaStream_t st, int in_sh, int out_sh,
                        const void* rowfilt, const BlockPtrs* ib, const BlockPtrs* ob) {
    if (rowfilt && inv) return cudaErrorInvalidValue;  // filter passes start with the forward transform
    // in == out is safe for the TMA kernel: every tile is read (prefetched)
    // by the CTA that later writes it, and no other CTA touches it
    if (use_tma_rows(prec, R, in_sh, out_sh)) {
        if (rowfilt)
            return real_in ? rows_tma_r<false, true, true>(R, in, out, batch, scale, tw, rowfilt, st)
                           : rows_tma_r<false, false, true>(R, in, out, batch, scale, tw, rowfilt, st);
        if (real_in) return rows_tma_r<false, true, false>(R, in, out, batch, scale, tw, nullptr, st);
        return inv ? rows_tma_r<true, false, false>(R, in, out, batch, scale, tw, nullptr, st)
                   : rows_tma_r<false, false, false>(R, in, out, batch, scale, tw, nullptr, st);
    }
    if (prec == 0) {
        if (rowfilt)
            return real_in ? rows_r<float, false, true, true>(R, in, out, batch, scale, tw, in_sh, out_sh, rowfilt, st, ib, ob)
                           : rows_r<float, false, false, true>(R, in, out, batch, scale, tw, in_sh, out_sh, rowfilt,
                                                               st, ib, ob);
        if (real_in) return rows_r<float, false, true, false>(R, in, out, batch, scale, tw, in_sh, out_sh, nullptr, st, ib, ob);
        return inv ? rows_r<float, true, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, nullptr, st, ib, ob)
                   : rows_r<float, false, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, nullptr, st, ib, ob);
    }
    if (real_in) return cudaErrorInvalidValue;
    if (rowfilt) return rows_r<double, false, false, true>(R, in, out, batch, scale, tw, in_sh, out_sh, rowfilt, st, ib, ob);
    return inv ? rows_r<double, true, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, nullptr, st, ib, ob)
               : rows_r<double, false, false, false>(R, in, out, batch, scale, tw, in_sh, out_sh, nullptr, st, ib, ob);
}

}  // namespace b200fft
