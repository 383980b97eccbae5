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
    using F = LineFFT<T, R, E, INV, 0, false, sizeof(T) == 4>;  // step twiddles by recurrence (c64)
    using G = PassPipeCfg<T, R, W>;
    constexpr int NT = W * F::TPL;
    constexpr int RS = NT / W;  // = TPL
    static_assert(NT % W == 0, "tile shape");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* stage0 = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    // short lines (TPL < 32): lines are the thread-fastest index, so a warp
    // touches 32 different lines at one offset and the odd line stride keeps
    // every exchange conflict-free (lane-fastest within a 4-/8-/16-thread line
    // put several lines in one bank group: 4-way conflicts, profiles/README.md)
    constexpr bool LF = F::TPL < 32;
    const int t = LF ? tid % W : tid / F::TPL, lt = LF ? tid / W : tid % F::TPL;
    const int tt = tid % W, r0 = tid / W;  // load / store mapping
    const int pr0 = pad16(r0);
    // padded slot of element r0 + it RS: compile-time offsets when RS is a
    // multiple of 16 (pad16(x + c) = pad16(x) + c + c / 16), else computed
    auto slot = [&](int it) { return (RS % 16 == 0) ? pr0 + it * (RS + RS / 16) : pad16(r0 + it * RS); };
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
            C* d = stage0 + buf * G::STAGE_ELEMS + tt * G::LS;
#pragma unroll
            for (int it = 0; it < R / RS; ++it) cp_async8(d + slot(it), s + (int64_t)it * RS * LR, true);
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
            C* d = sm + tt * G::LS;
            // W^{k (r0 + it RS)} = W^{k r0} (W^{k RS})^it: two table products
            C w = __ldg(wa);
            if (nhi > 1) w = cmul(w, __ldg(wb));
            C ws = __ldg(pa + (int64_t)RS * KLO + (kt & (KLO - 1)));
            if (nhi > 1) ws = cmul(ws, __ldg(pb + (int64_t)RS * nhi + (kt >> klo_sh)));
#pragma unroll
            for (int it = 0; it < R / RS; ++it) {
                d[slot(it)] = cmul_dir<INV>(d[slot(it)], w);
                w = cmul(w, ws);
            }
        }
        __syncthreads();
        C* line = sm + t * G::LS;
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
        const int bar = (!LF && F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
        F::run(v, line, lt, tw, bar);
        F::lsync(bar);
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
        __syncthreads();
        C* dst = out + bidx * L;
        if (Ns >= W) {  // consecutive threads -> consecutive k: W-element runs per q
            const int64_t jt = j0 + tt, kt = jt & (Ns - 1);
            C* d = dst + (jt - kt) * R + kt + (int64_t)r0 * Ns;
            const C* s = sm + tt * G::LS;
#pragma unroll
            for (int it = 0; it < R / RS; ++it) d[(int64_t)it * RS * Ns] = s[slot(it)];
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


// ---------------------------------------------------------------------------
// k_pass_tma: the same pass with the tile fetched by the TMA engine.  Each
// of the tile's R row segments (W consecutive butterflies = W x 8 B
// contiguous in HBM) is ONE cp.async.bulk into a dense [R][W] stage
// (2 stages, mbarrier completion), so the load side issues R instructions
// per tile instead of W R / 32 warp-wide LDGSTS (k_pass_pipe's stall was
// lg_throttle: the LSU queue full of 8-B copies).  After a stage lands,
// one smem pass moves it into the engine's padded line buffer, applying the
// pass twiddle on the way (consecutive threads = consecutive k: coalesced
// table reads, conflict-free odd line stride).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void mbar_init_pass(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_pass(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_pass(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PASS_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra PASS_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <typename T, int R, int W>
struct PassTmaCfg {
    static constexpr int LS = pad16c(R) + 1;
    static constexpr size_t STAGE_BYTES = sizeof(cpx<T>) * (size_t)R * W;  // dense [R][W]
    static constexpr size_t LINE_OFF = 2 * STAGE_BYTES;
    static constexpr size_t BAR_OFF = LINE_OFF + sizeof(cpx<T>) * (size_t)W * LS;
    static constexpr size_t SMEM_BYTES = BAR_OFF + 16;
    static constexpr uint32_t SEG_BYTES = (uint32_t)(W * sizeof(cpx<T>));
};

__device__ __forceinline__ void pass_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

template <typename T, int R, int E, int W, bool INV>
__global__ void __launch_bounds__(W*(R / E), 1)
    k_pass_tma(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t L, int64_t Ns, int64_t nlines,
               T scale, const cpx<T>* __restrict__ tw, const cpx<T>* __restrict__ pa, const cpx<T>* __restrict__ pb,
               int klo_sh) {
    using C = cpx<T>;
    using F = LineFFT<T, R, E, INV, 0, false, sizeof(T) == 4>;  // step twiddles by recurrence (c64)
    using G = PassTmaCfg<T, R, W>;
    constexpr int NT = W * F::TPL;
    static_assert((W * sizeof(C)) % 16 == 0, "bulk copies move multiples of 16 B");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* lines = reinterpret_cast<C*>(smem_raw + G::LINE_OFF);
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(smem_raw + G::BAR_OFF);
    const uint32_t st0 = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const int tid = threadIdx.x;
    // short lines (TPL < 32): lines are the thread-fastest index, so a warp
    // touches 32 different lines at one offset and the odd line stride keeps
    // every exchange conflict-free (lane-fastest within a 4-/8-/16-thread line
    // put several lines in one bank group: 4-way conflicts, profiles/README.md)
    constexpr bool LF = F::TPL < 32;
    const int t = LF ? tid % W : tid / F::TPL, lt = LF ? tid / W : tid % F::TPL;
    const int64_t LR = L / R;
    const int64_t ntiles = nlines / W;
    const int64_t KLO = (int64_t)1 << klo_sh;
    const int64_t nhi = Ns >> klo_sh;

    // the R row segments of `tile` -> stage s (thread r < R issues segment r;
    // thread 0 arms the barrier first, the others are ordered after it by
    // the __syncthreads that precedes every call)
    auto issue = [&](int64_t tile, int s) {
        if (tile >= ntiles) return;
        const int64_t gl0 = tile * W;
        const int64_t bidx = gl0 / LR;
        const int64_t j0 = gl0 - bidx * LR;
        for (int r = tid; r < R; r += NT)
            pass_bulk_g2s(st0 + (uint32_t)(s * G::STAGE_BYTES) + (uint32_t)r * G::SEG_BYTES,
                          in + bidx * L + j0 + (int64_t)r * LR, G::SEG_BYTES, bar0 + 8 * s);
    };
    if (tid == 0) {
        mbar_init_pass(bar0, 1);
        mbar_init_pass(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        if (blockIdx.x < ntiles) mbar_expect_tx_pass(bar0, (uint32_t)(R * G::SEG_BYTES));
        if (blockIdx.x + gridDim.x < ntiles) mbar_expect_tx_pass(bar0 + 8, (uint32_t)(R * G::SEG_BYTES));
    }
    __syncthreads();
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);

    for (int64_t i = 0;; ++i) {
        const int64_t tile = blockIdx.x + i * gridDim.x;
        if (tile >= ntiles) break;
        const int s = (int)(i & 1);
        mbar_wait_pass(bar0 + 8 * s, (uint32_t)((i >> 1) & 1));
        const int64_t gl0 = tile * W;
        const int64_t bidx = gl0 / LR;
        const int64_t j0 = gl0 - bidx * LR;
        // dense stage [r][tt] -> padded lines [tt][pad16(r)], x pass twiddle
        const C* sg = reinterpret_cast<const C*>(smem_raw + s * G::STAGE_BYTES);
        {
            const int tt = tid % W, r0 = tid / W;
            constexpr int RS = NT / W;
            const int64_t kt = (j0 + tt) & (Ns - 1);
            const C* wa = pa + (kt & (KLO - 1));
            const C* wb = pb + (kt >> klo_sh);
#pragma unroll 4
            for (int it = 0; it < R / RS; ++it) {
                const int r = r0 + it * RS;
                C a = sg[r * W + tt];
                if (Ns > 1) {
                    C w = __ldg(wa + (int64_t)r * KLO);
                    if (nhi > 1) w = cmul(w, __ldg(wb + (int64_t)r * nhi));
                    a = cmul_dir<INV>(a, w);
                }
                lines[tt * G::LS + pad16(r)] = a;
            }
        }
        __syncthreads();  // stage s consumed: refill it with the tile two ahead
        if (tid == 0 && tile + 2 * gridDim.x < ntiles) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            mbar_expect_tx_pass(bar0 + 8 * s, (uint32_t)(R * G::SEG_BYTES));
        }
        __syncthreads();
        issue(tile + 2 * gridDim.x, s);
        C* line = lines + t * G::LS;
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
        const int bar = (!LF && F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
        F::run(v, line, lt, tw, bar);
        F::lsync(bar);
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
        __syncthreads();
        C* dst = out + bidx * L;
        {
            constexpr int RS = NT / W;
            const int tt = tid % W, r0 = tid / W;
            if (Ns >= W) {  // consecutive threads -> consecutive k: W-element runs per q
                const int64_t jt = j0 + tt, kt = jt & (Ns - 1);
                C* d = dst + (jt - kt) * R + kt;
#pragma unroll 4
                for (int it = 0; it < R / RS; ++it) {
                    const int q = r0 + it * RS;
                    d[(int64_t)q * Ns] = lines[tt * G::LS + pad16(q)];
                }
            } else {  // Ns == 1: the tile's output is one contiguous block of W R elements
#pragma unroll 4
                for (int it = 0; it < (W * R) / NT; ++it) {
                    const int idx = tid + it * NT;
                    const int q = idx % R, tl = idx / R;
                    dst[(j0 + tl) * R + q] = lines[tl * G::LS + pad16(q)];
                }
            }
        }
        __syncthreads();  // the line buffer is rewritten by the next tile
    }
}

}  // namespace b200fft
