// fft_cols_pipe.cuh -- persistent, double-buffered column kernel (sm_100a).
//
// Same computation as k_cols (column DFTs of an [R][S] grid, MODE 2 = the
// fused forward -> filter -> inverse of the pipeline), but each CTA is
// persistent over column tiles and prefetches tile k+1 with cp.async
// (LDGSTS, asynchronous global -> shared copies straight into the padded
// line layout of the engine) while it transforms tile k in place.  The plain
// k_cols issues a tile's loads, waits for all of them, computes and stores:
// its warps mostly wait on long-scoreboard stalls (ncu, profiles/).
#pragma once
#include "fft_engine.cuh"

namespace b200fft {

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc, bool valid) {
    const uint32_t d = (uint32_t)__cvta_generic_to_shared(smem_dst);
    const int sz = valid ? 8 : 0;  // src-size 0 zero-fills
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(gsrc), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <typename T, int R, int W, int NS = 2>
struct ColsPipeCfg {
    static constexpr int LSC = cols_ls<T, R, W>();
    static constexpr size_t STAGE_ELEMS = (size_t)W * LSC;
    static constexpr size_t SMEM_BYTES = NS * STAGE_ELEMS * sizeof(cpx<T>);
};

// MODE 3 / 4 (the column direction of the 2D pipeline as a four-step over
// the column length N = N1 N2): MODE 3 is the
// forward column DFT (length R = N1, rows N2 M apart) followed by the
// twiddle W_N^{n2 u} (n2 = col / tdiv); MODE 4 multiplies the loaded
// element u by conj(W_N^{n2 u}) and runs the inverse DFT.  With kind 6,
// MODE 2's filter is g[img + n1 * u] (the frequency k1 + N1 k2 of the
// four-step's digit order).
// NS: ring of NS stages, NS - 1 tiles prefetched ahead (HBM bytes in
// flight per SM is what these streaming passes are bound by).
template <typename T, int R, int E, int W, int MODE, int NS = 2>
__global__ void __launch_bounds__(W*(R / E), 1)
    k_cols_pipe(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t S, int64_t nimg, T scale,
                const cpx<T>* __restrict__ tw, FilterArgs filt) {
    using C = cpx<T>;
    B200FFT_PDL_PROLOGUE();
    constexpr bool INV0 = (MODE == 1 || MODE == 4);
    // step twiddles: powers of one table entry for complex64 (TWREC), else
    // prefetched table entries
    constexpr bool TWR = sizeof(T) == 4;
    using F = LineFFT<T, R, E, INV0, 0, !TWR, TWR>;
    using FI = LineFFT<T, R, E, true, 0, !TWR, TWR>;
    using G = ColsPipeCfg<T, R, W, NS>;
    constexpr int NT = W * F::TPL;
    constexpr int LSC = G::LSC;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* stage0 = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    // short lines (TPL < 32): lines are the thread-fastest index, so a warp
    // touches 32 different lines at one offset and the odd line stride keeps
    // every exchange conflict-free (lane-fastest within a 4-/8-/16-thread line
    // put several lines in one bank group: 4-way conflicts, profiles/README.md)
    constexpr bool LF = F::TPL < 32;
    const int t = LF ? tid % W : tid / F::TPL, lt = LF ? tid / W : tid % F::TPL;
    const int64_t tiles_per_img = (S + W - 1) / W;
    const int64_t ntiles = tiles_per_img * nimg;

    auto prefetch = [&](int64_t tile, int buf) {
        if (tile < ntiles) {
            const int64_t img = tile / tiles_per_img;
            const int64_t s0 = (tile - img * tiles_per_img) * W;
            const C* src = in + img * (int64_t)R * S + s0;
            const int wv = (int)((S - s0) < W ? (S - s0) : W);
            C* sm = stage0 + buf * G::STAGE_ELEMS;
#pragma unroll
            for (int it = 0; it < (W * R) / NT; ++it) {
                const int idx = tid + it * NT;
                const int tt = idx % W, r = idx / W;
                const bool ok = tt < wv;
                cp_async8(sm + tt * LSC + pad16(r), ok ? src + (int64_t)r * S + tt : src, ok);
            }
        }
        cp_async_commit();  // one group per call (possibly empty): uniform wait counts
    };

#pragma unroll
    for (int j = 0; j < NS - 1; ++j) prefetch(blockIdx.x + (int64_t)j * gridDim.x, j);
    for (int64_t k = 0;; ++k) {
        const int64_t tile = blockIdx.x + k * gridDim.x;
        if (tile >= ntiles) break;
        const int buf = (int)(k % NS);
        prefetch(tile + (int64_t)(NS - 1) * gridDim.x, (int)((k + NS - 1) % NS));
        cp_async_wait<NS - 1>();  // this thread's copies of tile k have landed
        __syncthreads();          // ... and everyone else's
        const int64_t img = tile / tiles_per_img;
        const int64_t s0 = (tile - img * tiles_per_img) * W;
        const int wv = (int)((S - s0) < W ? (S - s0) : W);
        C* sm = stage0 + buf * G::STAGE_ELEMS;
        C* line = sm + t * LSC;
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
        if constexpr (MODE == 4) {  // conj(W^{n2 (lt + TPL m)}) = conj(W^{n2 lt} (W^{n2 TPL})^m)
            const int64_t n2 = (s0 + t) / filt.tdiv;
            const C* tl = reinterpret_cast<const C*>(filt.tw_l);
            C wm = __ldg(tl + n2 * lt);
            const C ws = __ldg(tl + n2 * F::TPL);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                v[F::pos_in(m)] = cmulc(v[F::pos_in(m)], wm);
                wm = cmul(wm, ws);
            }
        }
        const int bar = (!LF && F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
        F::run(v, line, lt, tw, bar);
        if constexpr (MODE == 3) {  // W^{n2 (lt + TPL m)} = W^{n2 lt} (W^{n2 TPL})^m
            const int64_t n2 = (s0 + t) / filt.tdiv;
            const C* tl = reinterpret_cast<const C*>(filt.tw_l);
            C wm = __ldg(tl + n2 * lt);
            const C ws = __ldg(tl + n2 * F::TPL);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                v[F::pos_out(m)] = cmul(v[F::pos_out(m)], wm);
                wm = cmul(wm, ws);
            }
        }
        if constexpr (MODE == 2) {
            C w[E];
            const int64_t col = s0 + t;
            if (filt.spec != nullptr && col < S) {
                float* sp = filt.spec + img * (int64_t)R * S + col;
#pragma unroll
                for (int m = 0; m < E; ++m)
                    sp[(int64_t)(lt + F::TPL * m) * S] = spec_mag(v[F::pos_out(m)], filt.spec_scale);
            }
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int64_t u = lt + F::TPL * m;
                const T hv = (filt.kind >= 6) ? fourstep_filter<T>(filt, img, u, col < S ? col : 0)
                                              : filter_value<T>(filt, u, col + filt.col_off);
                const T h = (col < S) ? hv * scale : (T)0;
                w[FI::pos_in(m)] = cscale(v[F::pos_out(m)], h);
            }
            FI::run(w, line, lt, tw, bar);
            F::lsync(bar);
#pragma unroll
            for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = w[FI::pos_out(m)];
        } else {
            F::lsync(bar);
#pragma unroll
            for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
        }
        __syncthreads();
        C* dst = out + img * (int64_t)R * S + s0;
#pragma unroll
        for (int it = 0; it < (W * R) / NT; ++it) {
            const int idx = tid + it * NT;
            const int tt = idx % W, r = idx / W;
            if (tt < wv) dst[(int64_t)r * S + tt] = sm[tt * LSC + pad16(r)];
        }
        __syncthreads();  // buffer `buf` is free for the prefetch NS tiles ahead
    }
    cp_async_wait<0>();
}

}  // namespace b200fft
