// fft_tma.cuh -- persistent, TMA-fed row FFT kernel (sm_100a).
//
// Same computation as k_rows (the paper's DFT, Eq. E2 / Eq. E3, on
// contiguous rows), but every CTA is persistent and keeps STAGES tiles of
// W rows in flight: one thread issues a bulk copy (cp.async.bulk, the TMA
// engine) of the next tiles into a ring of shared-memory stages, completing
// on per-stage mbarriers, while all threads run the Stockham steps IN PLACE
// in the current stage (unpadded, XOR-swizzled exchanges, LineFFT LAYOUT 1)
// and store the results straight from registers (coalesced).  HBM reads are
// therefore always outstanding, independent of the compute phase, instead of
// the load -> compute -> store convoy of one tile per CTA.
#pragma once
#include "fft_engine.cuh"

namespace b200fft {

__device__ __forceinline__ uint32_t smem_addr_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "TMA_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra TMA_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// Each row lands (one bulk copy per row) at the start of its padded line
// region (LS = pad16(R) + 2 slots: even, so every row start is 16-B
// aligned); step 0 reads it unpadded, every later exchange uses the padded
// index (LineFFT LAYOUT 0) in place.
template <typename T, int R, int W, bool REAL_IN, int STAGES>
struct RowsTmaCfg {
    static constexpr int LS = pad16c(R) + 2;
    static constexpr size_t STAGE_BYTES = sizeof(cpx<T>) * W * LS;
    static constexpr size_t SMEM_BYTES = STAGES * STAGE_BYTES + 8 * STAGES;
    static constexpr uint32_t ROW_IN_BYTES = (uint32_t)(R * (REAL_IN ? sizeof(float) : sizeof(cpx<T>)));
};

// One pass of tiles: the stage ring (STAGES stages of W lines at smem_raw,
// mbarriers at bar0) over tiles blockIdx.x, + gridDim.x, ...  The first
// STAGES tiles are issued by rows_tma_issue_first (thread 0) beforehand.
template <typename T, int R, int E, int W, bool REAL_IN, int STAGES>
__device__ __forceinline__ void rows_tma_issue(const void* in_, int64_t batch, unsigned char* smem_raw, uint32_t bar0,
                                               int64_t tile, int s) {
    using C = cpx<T>;
    using G = RowsTmaCfg<T, R, W, REAL_IN, STAGES>;
    const char* in = reinterpret_cast<const char*>(in_);
    const int64_t r0 = tile * W;
    const int64_t nr = (batch - r0) < W ? (batch - r0) : W;
    const uint32_t bar = bar0 + 8 * s;
    mbar_expect_tx(bar, (uint32_t)(nr * G::ROW_IN_BYTES));
    const uint32_t dst = smem_addr_u32(smem_raw + s * G::STAGE_BYTES);
    for (int64_t i = 0; i < nr; ++i)
        bulk_g2s(dst + (uint32_t)(i * G::LS * sizeof(C)), in + (r0 + i) * G::ROW_IN_BYTES, G::ROW_IN_BYTES, bar);
}

template <typename T, int R, int E, int W, bool REAL_IN, int STAGES>
__device__ __forceinline__ void rows_tma_issue_first(const void* in_, int64_t batch, unsigned char* smem_raw,
                                                     uint32_t bar0) {
    const int64_t ntiles = (batch + W - 1) / W;
    for (int s = 0; s < STAGES; ++s) {
        const int64_t tile = blockIdx.x + (int64_t)s * gridDim.x;
        if (tile < ntiles) rows_tma_issue<T, R, E, W, REAL_IN, STAGES>(in_, batch, smem_raw, bar0, tile, s);
    }
}

// TRANS: store the tile transposed, out[v][row] (leading dimension = batch),
// through the stage buffer so that the W rows of a tile form W-element runs
// -- the separable pipeline's passes then always read contiguous rows.
// PAIR (NEXT-3, real-to-real separable pipeline): each line is TWO real
// float32 rows a, b (the 2R floats a bulk copy of one complex row brings in)
// transformed as the complex row a + i b.  The row filter pass is a real
// operator when its filter is real and even (g[v] = g[R - v]: the Gaussian),
// so the result is L(a) + i L(b) exactly: real part = filtered a, imaginary
// part = filtered b, stored as the float pair (a', b') -- which, with TRANS,
// is the transposed real grid.  Half the lines, half the bytes of promoting
// each real row to complex.  PAIR = 2: the same, stored as the transposed
// COMPLEX grid (a', 0), (b', 0) -- the last pass of a real-input pipeline
// with complex output, whose exact result is real.
// xo: timing experiments only (wrong results): 1 = no FFT arithmetic, 2 = no stores.
template <typename T, int R, int E, int W, bool INV, bool REAL_IN, int STAGES, bool FILT, bool TRANS, int PAIR,
          int MLX = 0>
__device__ __forceinline__ void rows_tma_loop(const void* in_, cpx<T>* __restrict__ out, int64_t batch, T scale,
                                              const cpx<T>* __restrict__ tw, const T* __restrict__ rowfilt, int xo,
                                              unsigned char* smem_raw, uint32_t bar0) {
    using C = cpx<T>;
#ifndef B200FFT_ROWS_TWREC
#define B200FFT_ROWS_TWREC 1
#endif
    // step twiddles: prefetched table entries (default) or, with
    // B200FFT_ROWS_TWREC, powers of one entry (LineFFT TWREC)
    constexpr bool TWR = B200FFT_ROWS_TWREC != 0;
    using F = LineFFT<T, R, E, INV, 0, !TWR, TWR, MLX>;
    using G = RowsTmaCfg<T, R, W, REAL_IN, STAGES>;
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int64_t ntiles = (batch + W - 1) / W;

    for (int64_t k = 0;; ++k) {
        const int64_t tile = blockIdx.x + k * gridDim.x;
        if (tile >= ntiles) break;
        const int s = (int)(k % STAGES);
        mbar_wait(bar0 + 8 * s, (uint32_t)((k / STAGES) & 1));
        C* line = reinterpret_cast<C*>(smem_raw + s * G::STAGE_BYTES) + t * G::LS;
        C v[E];
        if constexpr (REAL_IN) {
            const float* fl = reinterpret_cast<const float*>(line);
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = mk((T)fl[lt + F::TPL * m], (T)0);
        } else if constexpr (PAIR) {
            const float* fl = reinterpret_cast<const float*>(line);
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = mk((T)fl[lt + F::TPL * m], (T)fl[R + lt + F::TPL * m]);
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[lt + F::TPL * m];
        }
        const int bar = (F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
        T sc = scale;
        if (!(xo & 1)) {
            F::run(v, line, lt, tw, bar);
            row_filter_pass<T, R, E, FILT, 0, !TWR, TWR, MLX>(v, line, lt, tw, rowfilt, sc, bar);
        }
        const int64_t row = tile * W + t;
        if (xo & 2) {
            if (v[0].x == (T)1.2345e-30) out[0] = v[0];
        } else if constexpr (TRANS) {
            F::lsync(bar);
#pragma unroll
            for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], sc);
            __syncthreads();
            const C* sg = reinterpret_cast<const C*>(smem_raw + s * G::STAGE_BYTES);
            const int64_t r0 = tile * W;
            constexpr int NT = W * F::TPL;
#pragma unroll 4
            for (int it = 0; it < (W * R) / NT; ++it) {
                const int idx = tid + it * NT;
                const int tt = idx % W, vv = idx / W;
                if (r0 + tt < batch) {
                    if constexpr (PAIR == 2) {
                        const C x = sg[tt * G::LS + pad16(vv)];
                        reinterpret_cast<float4*>(out)[(int64_t)vv * batch + r0 + tt] =
                            make_float4((float)x.x, 0.f, (float)x.y, 0.f);
                    } else {
                        out[(int64_t)vv * batch + r0 + tt] = sg[tt * G::LS + pad16(vv)];
                    }
                }
            }
        } else if (row < batch) {
            C* o = out + row * R + lt;
#pragma unroll
            for (int m = 0; m < E; ++m) o[F::TPL * m] = cscale(v[F::pos_out(m)], sc);
        }
        __syncthreads();  // every thread is done with stage s
        if (tid == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const int64_t nt = blockIdx.x + (k + STAGES) * gridDim.x;
            if (nt < ntiles) rows_tma_issue<T, R, E, W, REAL_IN, STAGES>(in_, batch, smem_raw, bar0, nt, s);
        }
    }
}

template <typename T, int R, int E, int W, bool INV, bool REAL_IN, int STAGES, bool FILT = false, bool TRANS = false,
          int PAIR = 0, int MINB = 1>
__global__ void __launch_bounds__(W*(R / E), MINB)
    k_rows_tma(const void* __restrict__ in_, cpx<T>* __restrict__ out, int64_t batch, T scale,
               const cpx<T>* __restrict__ tw, const T* __restrict__ rowfilt, int xo = 0) {
    using G = RowsTmaCfg<T, R, W, REAL_IN, STAGES>;
    static_assert(R >= 256 && (R * sizeof(cpx<T>)) % 16 == 0, "bulk copies need >= 16 B rows");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t bar0 = smem_addr_u32(smem_raw + STAGES * G::STAGE_BYTES);
    // programmatic dependent launch: when this launch overlaps the tail of
    // the previous kernel (the second pass of a pipeline), wait for that
    // kernel's results before the first load; let the next one launch early
    // (both no-ops for an ordinary launch)
    B200FFT_PDL_PROLOGUE();
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        rows_tma_issue_first<T, R, E, W, REAL_IN, STAGES>(in_, batch, smem_raw, bar0);
    }
    __syncthreads();
    rows_tma_loop<T, R, E, W, INV, REAL_IN, STAGES, FILT, TRANS, PAIR>(in_, out, batch, scale, tw, rowfilt, xo,
                                                                         smem_raw, bar0);
}

// ---------------------------------------------------------------------------
// k_rows_tma_g: long natural rows (one row per stage) processed by NG
// independent thread groups of R/E threads each, E values per thread (the
// 8192-point rows of C4: E = 32, two groups of 256 threads, radix-32 steps
// (MLX 5: 8192 = 32 x 32 x 8, two exchanges per transform instead of the
// three of radix 16): the row filter pass 430 -> 355 us, C4 0.897 -> 0.832
// ms; the same groups with radix-16 steps measured no gain, a 33-slot
// padding that removes the first write's 2-way bank conflicts measured
// equal (it spills)).  Group g takes the CTA's tiles k = g, g + NG,
// ... from the shared ring of STAGES stages; its steps synchronise on its own
// named barrier (1 + g), so one group's exchanges and barriers overlap the
// other's arithmetic, and each thread has twice the independent work of the
// one-group E = 16 form.  The group that finishes a stage refills it with
// the tile STAGES positions later (which another group may consume: the
// per-stage mbarrier phase orders them).  Natural stores (no TRANS / PAIR).
// ---------------------------------------------------------------------------
template <typename T, int R, int E, int NG, bool INV, int STAGES, bool FILT, int MLX = 0>
__global__ void __launch_bounds__(NG*(R / E), 1)
    k_rows_tma_g(const void* __restrict__ in_, cpx<T>* __restrict__ out, int64_t batch, T scale,
                 const cpx<T>* __restrict__ tw, const T* __restrict__ rowfilt) {
    using C = cpx<T>;
    using F = LineFFT<T, R, E, INV, 0, false, true, MLX>;
    using G = RowsTmaCfg<T, R, 1, false, STAGES>;
    static_assert(F::TPL % 32 == 0 && NG <= 15, "whole warps per group, named barriers 1..NG");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t bar0 = smem_addr_u32(smem_raw + STAGES * G::STAGE_BYTES);
    B200FFT_PDL_PROLOGUE();
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        rows_tma_issue_first<T, R, E, 1, false, STAGES>(in_, batch, smem_raw, bar0);
    }
    __syncthreads();
    const int g = threadIdx.x / F::TPL, lt = threadIdx.x % F::TPL;
    const int bar = 1 + g;
    for (int64_t k = g;; k += NG) {
        const int64_t row = blockIdx.x + k * gridDim.x;
        if (row >= batch) break;
        const int s = (int)(k % STAGES);
        mbar_wait(bar0 + 8 * s, (uint32_t)((k / STAGES) & 1));
        C* line = reinterpret_cast<C*>(smem_raw + s * G::STAGE_BYTES);
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[lt + F::TPL * m];
        F::run(v, line, lt, tw, bar);
        T sc = scale;
        row_filter_pass<T, R, E, FILT, 0, false, true, MLX>(v, line, lt, tw, rowfilt, sc, bar);
        C* o = out + row * R + lt;
#pragma unroll
        for (int m = 0; m < E; ++m) o[F::TPL * m] = cscale(v[F::pos_out(m)], sc);
        F::lsync(bar);  // the group is done with stage s
        if (lt == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const int64_t nk = k + STAGES;
            if (blockIdx.x + nk * gridDim.x < batch)
                rows_tma_issue<T, R, E, 1, false, STAGES>(in_, batch, smem_raw, bar0, blockIdx.x + nk * gridDim.x, s);
        }
    }
}

// ---------------------------------------------------------------------------
// k_rows_tma2: BOTH passes of the separable real-pair pipeline (C3's shape,
// square R x R grids, R <= 2048) in ONE cooperative launch: pass 1 = the
// row filter pass over the input's real-row pairs, stored transposed into
// the intermediate `mid` (PAIR 1: float pairs); a grid-wide barrier; pass 2
// = the row filter pass over the transposed grid's row pairs, stored
// transposed into `out` (PAIR2 = 2: complex (a, 0), (b, 0); 1: real pairs).
// One launch instead of two saves the second launch's ramp and tail (the
// C3 breakdown: ~15 us of the 40 were launch + first-load latency).
// Grid barrier without host-side state (so a CUDA-graph replay of a launch
// is correct): *gbar counts arrivals and only grows; thread 0 of every CTA
// reads it at kernel start -- before its own arrival, so between k grid and
// k grid + grid - 1 when k launches (of this plan, same grid) completed --
// and waits for target = (k + 1) grid.  At the barrier it releases the
// CTA's pass-1 stores at gpu scope (bar.sync + fence.acq_rel.gpu:
// cumulative), arrives, and polls (acquire); then a proxy fence orders the
// generic-proxy stores before the TMA (async proxy) reads of pass 2.  All
// CTAs are co-resident (cooperative launch); launches of one plan are
// stream-ordered, so they never share the counter at once.  (A host-passed
// target -- the earlier form -- is frozen by graph capture: a replay would
// pass the barrier early.)
// ---------------------------------------------------------------------------
template <int R, int E, int W, int STAGES, int PAIR2, int MLX = 0>
__global__ void __launch_bounds__(W*(R / E), 1)
    k_rows_tma2(const void* __restrict__ in_, float2* __restrict__ mid, void* __restrict__ out_, int64_t lines,
                const float2* __restrict__ tw, float scale1, const float* __restrict__ filt1, float scale2,
                const float* __restrict__ filt2, unsigned long long* gbar, int xo) {
    using G = RowsTmaCfg<float, R, W, false, STAGES>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const uint32_t bar0 = smem_addr_u32(smem_raw + STAGES * G::STAGE_BYTES);
    const uint32_t bar1 = bar0 + 8 * STAGES;
    unsigned long long target = 0;  // thread 0: this launch's barrier count
    if (threadIdx.x == 0) {
        unsigned long long c0;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];\n" : "=l"(c0) : "l"(gbar) : "memory");
        target = (c0 / gridDim.x + 1) * (unsigned long long)gridDim.x;
        for (int s = 0; s < 2 * STAGES; ++s) mbar_init(bar0 + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        rows_tma_issue_first<float, R, E, W, false, STAGES>(in_, lines, smem_raw, bar0);
    }
    __syncthreads();
    rows_tma_loop<float, R, E, W, false, false, STAGES, true, true, 1, MLX>(in_, mid, lines, scale1, tw, filt1, xo,
                                                                           smem_raw, bar0);
    // ---- grid barrier (the loop ended with a __syncthreads) ----
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
        asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;\n" ::"l"(gbar) : "memory");
        unsigned long long v;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];\n" : "=l"(v) : "l"(gbar) : "memory");
            if (v >= target) break;
            __nanosleep(64);
        }
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        rows_tma_issue_first<float, R, E, W, false, STAGES>(mid, lines, smem_raw, bar1);
    }
    __syncthreads();
    rows_tma_loop<float, R, E, W, false, false, STAGES, true, true, PAIR2, MLX>(
        mid, reinterpret_cast<float2*>(out_), lines, scale2, tw, filt2, xo, smem_raw, bar1);
}

}  // namespace b200fft
