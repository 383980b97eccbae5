// fft_pass_pipe.cuh -- persistent, double-buffered global Stockham pass
// (kernel family C of fft_engine.cuh, sm_100a).
//
// Same computation as k_pass (one radix-R pass of a multi-pass transform of
// length L = 2^m > 8192, the DFT of Eq. E2 / E3, split
// into passes by the index map of Stockham's autosort):
//   v[r] = a[j + r L/R] * W_{Ns R}^{k r},  k = j mod Ns
//   b[(j - k) R + k + q Ns] = scale * sum_r v[r] W_R^{r q}
// but each CTA is persistent over tiles of W consecutive butterflies j and
// prefetches tile i+1 with cp.async (global -> shared, straight into the
// padded line layout) while it transforms tile i.  The pass twiddle is
// applied in shared memory right after the tile lands, in the load mapping
// (consecutive threads = consecutive k), so its table reads stay coalesced.
// k_pass issues a tile's loads, waits for them and only then computes: its
// warps mostly sit on long-scoreboard stalls (profiles/).
#pragma once
#include "fft_cols_pipe.cuh"

namespace b200fft {

template <typename T, int R, int W>
struct PassPipeCfg {
    static constexpr int LS = pad16c(R) + 1;
    static constexpr size_t STAGE_ELEMS = (size_t)W * LS;
    static constexpr size_t SMEM_BYTES = 2 * STAGE_ELEMS * sizeof(cpx<T>);
};

template <typename T, int R, int E, int W, bool INV>
__global__ void __launch_bounds__(W*(R / E), 1)
    k_pass_pipe(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t L, int64_t Ns, int64_t nlines,
                T scale, const cpx<T>* __restrict__ tw, const cpx<T>* __restrict__ pa,
                const cpx<T>* __restrict__ pb, int klo_sh) {
    using C = cpx<T>;
    using F = LineFFT<T, R, E, INV>;
    using G = PassPipeCfg<T, R, W>;
    constexpr int NT = W * F::TPL;
    constexpr int RS = NT / W;  // = TPL
    static_assert(NT % W == 0 && RS % 16 == 0, "tile shape");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* stage0 = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int tt = tid % W, r0 = tid / W;  // load / store mapping
    const int pr0 = pad16(r0);
    const int64_t LR = L / R;
    const int64_t ntiles = nlines / W;
    const int64_t KLO = (int64_t)1 << klo_sh;
    const int64_t nhi = Ns >> klo_sh;

    auto prefetch = [&](int64_t tile, int buf) {
        if (tile < ntiles) {
            const int64_t gl0 = tile * W;
            const int64_t bidx = gl0 / LR;
            const int64_t jt = gl0 - bidx * LR + tt;
            const C* s = in + bidx * L + jt + (int64_t)r0 * LR;
            C* d = stage0 + buf * G::STAGE_ELEMS + tt * G::LS + pr0;
#pragma unroll
            for (int it = 0; it < R / RS; ++it) cp_async8(d + it * (RS + RS / 16), s + (int64_t)it * RS * LR, true);
        }
        cp_async_commit();
    };

    prefetch(blockIdx.x, 0);
    for (int64_t i = 0;; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) break;
        const int buf = (int)(i & 1);
        prefetch(tile + gridDim.x, buf ^ 1);
        cp_async_wait<1>();
        const int64_t gl0 = tile * W;
        const int64_t bidx = gl0 / LR;
        const int64_t j0 = gl0 - bidx * LR;
        C* sm = stage0 + buf * G::STAGE_ELEMS;
        if (Ns > 1) {  // pass twiddle on this thread's own landed elements
            const int64_t kt = (j0 + tt) & (Ns - 1);
            const C* wa = pa + (int64_t)r0 * KLO + (kt & (KLO - 1));
            const C* wb = pb + (int64_t)r0 * nhi + (kt >> klo_sh);
            C* d = sm + tt * G::LS + pr0;
#pragma unroll
            for (int it = 0; it < R / RS; ++it) {
                C w = __ldg(wa + (int64_t)it * RS * KLO);
                if (nhi > 1) w = cmul(w, __ldg(wb + (int64_t)it * RS * nhi));
                d[it * (RS + RS / 16)] = cmul_dir<INV>(d[it * (RS + RS / 16)], w);
            }
        }
        __syncthreads();
        C* line = sm + t * G::LS;
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
        const int bar = (F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
        F::run(v, line, lt, tw, bar);
        F::lsync(bar);
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
        __syncthreads();
        C* dst = out + bidx * L;
        if (Ns >= W) {  // consecutive threads -> consecutive k: W-element runs per q
            const int64_t jt = j0 + tt, kt = jt & (Ns - 1);
            C* d = dst + (jt - kt) * R + kt + (int64_t)r0 * Ns;
            const C* s = sm + tt * G::LS + pr0;
#pragma unroll
            for (int it = 0; it < R / RS; ++it) d[(int64_t)it * RS * Ns] = s[it * (RS + RS / 16)];
        } else {  // Ns == 1: the tile's output is one contiguous block of W R elements
#pragma unroll
            for (int it = 0; it < (W * R) / NT; ++it) {
                const int idx = tid + it * NT;
                const int q = idx % R, tl = idx / R;
                const int64_t j = j0 + tl, k = j & (Ns - 1);
                dst[(j - k) * R + k + (int64_t)q * Ns] = sm[tl * G::LS + pad16(q)];
            }
        }
        __syncthreads();  // buffer `buf` is free for the prefetch two tiles ahead
    }
    cp_async_wait<0>();
}

}  // namespace b200fft
