// fft_c2.cuh -- the 65536-point complex64 transform of C2 (BASELINE
// configs[1]) in ONE HBM pass: a persistent task pipeline through an
// L2-resident ring.
//
// What is computed: the DFT of Eq. E2 (Sec. 2) with its
// 1/N, or the unscaled inverse of Eq. E3 / Sec. 3, by
// the four-step split n = n1 + 256 n2, k = k2 + 256 k1 (N = 65536):
//   A(b, p): columns n1 in [16p, 16p + 16) of transform b: 256-point DFTs over
//            n2 -> k2, twiddle W_N^{n1 k2}, Y[k2][n1] -> ring slot b % ring
//   B(b, p): rows k2 in [16p, 16p + 16) of Y(b): 256-point DFTs over n1 -> k1,
//            scale, X[k2 + 256 k1] -> HBM
// The same sums as the paper's radix-2 tree, reassociated.
//
// Scheduling (deadlock-free): a persistent
// cooperative grid walks one global task order A(0..D-1) | A(D) B(0) |
// A(D+1) B(1) | ... | B(batch-D..); per-transform counters done_a (A parts
// whose Y rows are in the ring) and done_b (B parts that have read theirs)
// order B(b) after A(b) and the reuse of a ring slot after its B parts, with
// release / acquire at gpu scope.  Waits only ever point back in the order.
#pragma once
#include <cuda.h>

#include "fft_engine.cuh"

namespace b200fft {

struct AbCtl {
    int* done_a;  // [batch] A parts of transform b whose Y rows are in the ring
    int* done_b;  // [batch] B parts of transform b that have read their Y rows
    int D, ring;  // dependency distance (transforms), ring slots
};

// ---- mbarrier / bulk-copy / TMA primitives (sm_90+ PTX) ------------------
__device__ __forceinline__ void bk_mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void bk_arrive_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bk_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void bk_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "BK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra BK_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bk_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ int bk_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void bk_red_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

namespace tmaops {
__device__ __forceinline__ void load3(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, uint32_t bar,
                                      uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;\n" ::"r"(dst),
        "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void store3(const CUtensorMap* map, int c0, int c1, int c2, uint32_t src, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;\n" ::"l"(
            map),
        "r"(c0), "r"(c1), "r"(c2), "r"(src), "l"(pol)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void prefetch3(const CUtensorMap* map, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];\n" ::"l"(map), "r"(c0), "r"(c1),
                 "r"(c2)
                 : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
    return p;
}
}  // namespace tmaops

// position i of the global task order -> (is B, transform b, part p)
__device__ __forceinline__ void ab_decode(int64_t i, int64_t batch, int64_t Dp, bool& isb, int64_t& b, int& part) {
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp);
    if (i < n1t) {
        isb = false;
        b = i / 16;
        part = (int)(i % 16);
    } else if (i < n1t + n2t) {
        const int64_t j = i - n1t, r = j % 32;
        isb = r >= 16;
        b = Dp + j / 32 - (isb ? Dp : 0);
        part = (int)(r % 16);
    } else {
        const int64_t j = i - n1t - n2t;
        isb = true;
        b = batch - Dp + j / 16;
        part = (int)(j % 16);
    }
}

// ---------------------------------------------------------------------------
// k_ab_ws: warp-specialised TMA form.  8 compute warps + 1 producer warp per
// CTA, 3 CTAs/SM, NS = 2 smem stages of 32 KiB used IN PLACE for a whole task:
// the TMA box lands in the stage (A: the dense [256 n2][16 n1] column box;
// B: the 16 contiguous 2 KiB Y rows), the engine exchanges inside it (A:
// LineFFT LAYOUT 2 = 16 interleaved lines; B: XOR-swizzled rows, LAYOUT 1),
// the results are written back into it as the output box (B with the 128-B
// TMA swizzle) and the producer stores it with one TMA instruction.  The
// producer alone issues loads (with the B dependency wait), stores, waits
// for their completion and signals done_a / done_b, so the compute warps
// only ever wait on the stage's full barrier and their named barrier.
// opts: bits 4..6 = L2 prefetch distance (tasks) of a later A tile (1 = best
// measured); bit 7 = the A twiddles W_N^{n1 (l + 16 m)} as W_N^{n1 l}
// (W_N^{16 n1})^m from two table entries (fp32, ~15 ulp) instead of 16 loads.
// ---------------------------------------------------------------------------
struct AbWsCfg {
    static constexpr int NS = 2;
    static constexpr size_t STAGE = 16 * 256 * 8;
    static constexpr size_t BAR_OFF = NS * STAGE;  // full[NS], comp[NS]
    static constexpr size_t SMEM = BAR_OFF + 16 * NS;
};

template <bool INV>
__global__ void __launch_bounds__(288, 3)
    k_ab_ws(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yst,
            const __grid_constant__ CUtensorMap map_yld, const __grid_constant__ CUtensorMap map_out, int64_t batch,
            float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbCtl ctl, int opts) {
    using G = AbWsCfg;
    constexpr int NS = G::NS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, comp0 = full0 + 8 * NS;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t ntasks = 32 * batch;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            bk_mbar_init(full0 + 8 * s, 1);
            bk_mbar_init(comp0 + 8 * s, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t my_tasks = ntasks > blockIdx.x ? (ntasks - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid >= 256) {  // ---- producer warp: lane 0 drives the TMA ----
        if (tid != 256) return;
        const uint64_t pol_stream = tmaops::policy_evict_first();
        const uint64_t pol_keep = tmaops::policy_evict_last();
        auto load = [&](int64_t k) {
            bool isb;
            int64_t b;
            int part;
            ab_decode(blockIdx.x + k * gridDim.x, batch, Dp, isb, b, part);
            const int s = (int)(k % NS);
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
            if (!isb) {
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_x, part * 16, 0, (int)b, bar, pol_stream);
            } else {
                while (bk_ld_acquire(ctl.done_a + b) < 16) __nanosleep(32);
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_yld, 0, part * 16, (int)(b % ctl.ring), bar, pol_keep);
            }
        };
        auto store = [&](int64_t k) {  // task k's outputs are in its stage
            bool isb;
            int64_t b;
            int part;
            ab_decode(blockIdx.x + k * gridDim.x, batch, Dp, isb, b, part);
            const int s = (int)(k % NS);
            bk_wait(comp0 + 8 * s, (uint32_t)((k / NS) & 1));
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
            if (!isb) {
                if (b >= ctl.ring)  // the slot's previous transform fully read
                    while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(32);
                tmaops::store3(&map_yst, part * 16, 0, (int)(b % ctl.ring), st, pol_keep);
                bk_store_wait_all();  // Y rows written: signal now (B tasks of other CTAs wait on it)
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + b, 1);
            } else {
                bk_red_release(ctl.done_b + b, 1);  // its Y rows were loaded before its compute
                tmaops::store3(&map_out, part * 16, 0, (int)b, st, pol_stream);
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // stage reusable
            }
        };
        const int pf = (opts >> 4) & 7;  // L2 prefetch distance (tasks) for A tiles, 0 = off
        for (int64_t k = 0; k < my_tasks; ++k) {
            if (k >= NS) store(k - NS);
            load(k);
            if (pf && k + pf < my_tasks) {  // warm L2 with a later A task's HBM tile
                bool pb;
                int64_t pbb;
                int ppart;
                ab_decode(blockIdx.x + (k + pf) * gridDim.x, batch, Dp, pb, pbb, ppart);
                if (!pb) tmaops::prefetch3(&map_x, ppart * 16, 0, (int)pbb);
            }
        }
        for (int64_t k = (my_tasks > NS ? my_tasks - NS : 0); k < my_tasks; ++k) store(k);
        bk_store_wait_all();
        return;
    }

    // ---- compute warps (256 threads) ----
    using FA = LineFFT<float, 256, 16, INV, 2, false, true>;
    using FB = LineFFT<float, 256, 16, INV, 1, false, true>;
    for (int64_t k = 0; k < my_tasks; ++k) {
        bool isb;
        int64_t b;
        int part;
        ab_decode(blockIdx.x + k * gridDim.x, batch, Dp, isb, b, part);
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        float2 v[16];
        if (!isb) {
            const int t = tid % 16, l = tid / 16;  // line = column n1 = 16 part + t
            const float2* tp = tw4 + (int64_t)l * 256 + part * 16 + t;
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FA::pos_in(m)] = line[FA::bpos(l, m)];
            FA::run(v, line, l, tw256, -256);
            FA::lsync(-256);
            if (opts & 128) {
                // W_N^{n1 (l + 16 m)} = W_N^{n1 l} (W_N^{16 n1})^m
                float2 wm = __ldg(tp);
                const float2 ws = __ldg(tw4 + (int64_t)16 * 256 + part * 16 + t);
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    line[(l + 16 * m) * 16] = cmul_dir<INV>(v[FA::pos_out(m)], wm);
                    wm = cmul(wm, ws);
                }
            } else {
#pragma unroll
                for (int m = 0; m < 16; ++m)
                    line[(l + 16 * m) * 16] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tp + (int64_t)m * 16 * 256));
            }
        } else {
            const int t = tid / 16, l = tid % 16;  // line = row k2 = 16 part + t of Y
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t * 256;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FB::pos_in(m)] = line[l + 16 * m];  // as landed (unswizzled)
            FB::run(v, line, l, tw256, -256);
            FB::lsync(-256);
            char* sb = reinterpret_cast<char*>(st);  // X box [k1][16 k2], 128-B swizzle
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int k1 = l + 16 * m;
                *reinterpret_cast<float2*>(sb + k1 * 128 + (((t >> 1) ^ (k1 & 7)) << 4) + ((t & 1) << 3)) =
                    cscale(v[FB::pos_out(m)], scale);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bk_arrive(comp0 + 8 * s);
    }
}

}  // namespace b200fft
