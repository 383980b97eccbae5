// fft_abbulk.cuh -- the 65536-point transform (C2) as independent 16-line
// tasks moved entirely by the TMA engine (sm_100a bulk copies), variant 40.
//
// Same four-step as fft_cluster.cuh (the DFT of Eq. E2 / E3, PAPER.md
// P:78-95, by the index split n = n1 + 256 n2, k = k2 + 256 k1):
//   A(b, p): columns n1 in [16p, 16p + 16) of transform b: 256-point DFTs
//            over n2, twiddle W_N^{n1 k2}, Y[k2][n1] -> an L2-resident ring
//   B(b, p): rows k2 in [16p, 16p + 16) of Y(b): 256-point DFTs over n1,
//            scale, X[k2 + 256 k1] -> HBM
// Every byte moves by cp.async.bulk: a task's 256 row segments of 128 B
// (A input, A / B output) or 16 rows of 2 KiB (B input) are one bulk copy per
// thread, loads completing on a per-stage mbarrier, stores tracked by bulk
// async-groups.  So no thread waits on a global load: a CTA transforms task
// i from smem while task i + 1's bytes land in the other stage.  Persistent
// grid (2 CTAs/SM), fixed global task order A(0..D-1) | A(D) B(0) | ...,
// counters done_a / done_b with release / acquire at gpu scope.  Waits are
// only ever on tasks earlier in the order (16 D >= 2 grid + margin), so
// co-resident CTAs (cooperative launch) cannot deadlock.
#pragma once
#include <cuda.h>

#include "fft_engine.cuh"

namespace b200fft {

struct AbBulkCtl {
    int* done_a;  // [batch] A parts of transform b whose Y rows are in L2
    int* done_b;  // [batch] B parts of transform b that have read their Y rows
    int D, ring;
};

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
__device__ __forceinline__ void bk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void bk_store(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void bk_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ int bk_ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// wait until *p >= target: relaxed polling (no L1 invalidation per poll --
// an acquire load invalidates the SM's L1, twiddle tables included, every
// iteration), then one acquire fence
__device__ __forceinline__ void bk_wait_count(const int* p, int target) {
    int v;
    for (;;) {
        asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
        if (v >= target) break;
        __nanosleep(32);
    }
    asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
}
__device__ __forceinline__ void bk_red_release(int* p, int v) {
    asm volatile("red.release.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

struct AbBulkCfg {
    static constexpr int RS = 18;                           // A tile / staging row stride (16 + 2, 16-B rows)
    static constexpr int BS = 258;                          // B tile row stride (256 + 2)
    static constexpr int LS = pad16c(256) + 1;              // engine line stride
    static constexpr size_t STAGE = 256 * RS * 8;           // >= 16 * BS * 8
    static constexpr size_t LINES = 16 * LS * 8;            // engine exchange buffer, also the output staging
    static constexpr size_t LINES_PAD = (LINES > STAGE ? LINES : STAGE);
    static constexpr size_t BAR_OFF = 2 * STAGE + LINES_PAD;
    static constexpr size_t SMEM = BAR_OFF + 16;
};

template <bool INV>
__global__ void __launch_bounds__(256, 2)
    k_ab_bulk(const float2* __restrict__ in, float2* __restrict__ out, float2* __restrict__ ring, int64_t batch,
              float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbBulkCtl ctl) {
    using G = AbBulkCfg;
    using F = LineFFT<float, 256, 16, INV>;
    constexpr int64_t N = 65536;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    float2* lines = reinterpret_cast<float2*>(smem_raw + 2 * G::STAGE);
    const uint32_t lines_s = s_base + (uint32_t)(2 * G::STAGE);
    const uint32_t bar0 = s_base + (uint32_t)G::BAR_OFF;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp), ntasks = 32 * batch;

    auto decode = [&](int64_t i, bool& isb, int64_t& b, int& part) {
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
    };
    // all threads: task i's input -> stage s (one bulk copy per row segment)
    auto issue = [&](int64_t i, int s) {
        if (i >= ntasks) return;
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
        const uint32_t bar = bar0 + 8 * s;
        if (!isb) {  // row n2 = tid, columns [16 part, +16) of transform b
            bk_arrive_expect(bar, 128);
            bk_load(st + (uint32_t)(tid * G::RS * 8), in + b * N + (int64_t)tid * 256 + part * 16, 128, bar);
        } else {  // rows k2 = 16 part + tid (tid < 16) of Y(b), once A(b) is complete
            if (tid == 0) {
                while (bk_ld_acquire(ctl.done_a + b) < 16) __nanosleep(64);
            }
            __syncthreads();
            if (tid < 16) {
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, 2048);
                bk_load(st + (uint32_t)(tid * G::BS * 8), ring + (b % ctl.ring) * N + (int64_t)(part * 16 + tid) * 256,
                        2048, bar);
            } else {
                bk_arrive(bar);
            }
        }
    };

    if (tid == 0) {
        bk_mbar_init(bar0, 256);
        bk_mbar_init(bar0 + 8, 256);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    issue(blockIdx.x, 0);
    issue(blockIdx.x + gridDim.x, 1);

    int64_t prev_a = -1;  // transform of this CTA's last A task, signalled one task late
    for (int64_t k = 0;; ++k) {
        const int64_t i = blockIdx.x + k * gridDim.x;
        if (i >= ntasks) break;
        const int s = (int)(k & 1);
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        // the previous task's bulk stores (from the staging = line buffer) are
        // complete: the buffer is reusable and an A task's Y is in L2
        bk_store_wait_all();
        bk_wait(bar0 + 8 * s, (uint32_t)((k >> 1) & 1));
        const float2* st = reinterpret_cast<const float2*>(smem_raw + s * G::STAGE);
        float2 v[16];
        // A: lines = columns, thread-fastest (t = tid % 16); B: lines = rows of
        // Y, lane-fastest within a line (conflict-free reads of the 2 KiB rows)
        const int t = isb ? tid / 16 : tid % 16, l = isb ? tid % 16 : tid / 16;
        if (!isb) {
#pragma unroll
            for (int m = 0; m < 16; ++m) v[F::pos_in(m)] = st[(l + 16 * m) * G::RS + t];
        } else {
#pragma unroll
            for (int m = 0; m < 16; ++m) v[F::pos_in(m)] = st[t * G::BS + l + 16 * m];
        }
        __syncthreads();  // stage s consumed; every thread's previous stores are done
        if (tid == 0) {
            if (prev_a >= 0) {
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + prev_a, 1);
            }
            if (isb) bk_red_release(ctl.done_b + b, 1);  // this B part has read its Y rows
        }
        prev_a = -1;
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        issue(i + 2 * gridDim.x, s);
        F::run(v, lines + t * G::LS, l, tw256);
        __syncthreads();  // the line buffer becomes the output staging
        float2* stg = lines;
        if (!isb) {
            const int n1 = part * 16 + t;
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int k2 = l + 16 * m;
                stg[k2 * G::RS + t] = cmul_dir<INV>(v[F::pos_out(m)], __ldg(tw4 + (int64_t)k2 * 256 + n1));
            }
        } else {
#pragma unroll
            for (int m = 0; m < 16; ++m) stg[(l + 16 * m) * G::RS + t] = cscale(v[F::pos_out(m)], scale);
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        if (!isb && b >= ctl.ring && tid == 0) {  // ring slot free (its previous B parts have read it)
            while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(64);
        }
        __syncthreads();
        if (!isb) {  // Y[k2 = tid][16 part .. +16]
            bk_store(ring + (b % ctl.ring) * N + (int64_t)tid * 256 + part * 16, lines_s + (uint32_t)(tid * G::RS * 8),
                     128);
            prev_a = b;
        } else {  // X[k2 + 256 k1], k1 = tid, k2 in [16 part, +16)
            bk_store(out + b * N + (int64_t)tid * 256 + part * 16, lines_s + (uint32_t)(tid * G::RS * 8), 128);
        }
    }
    bk_store_wait_all();
    __syncthreads();
    if (tid == 0 && prev_a >= 0) {
        asm volatile("fence.proxy.async.global;\n" ::: "memory");
        bk_red_release(ctl.done_a + prev_a, 1);
    }
}


// ---------------------------------------------------------------------------
// Variant 41: the same tasks with every tile moved by ONE tensor-map TMA
// instruction issued by thread 0 (2D boxes of 16 x 256 elements; the B
// output box is stored with the 128-B swizzle so the lane-fastest staging
// writes stay nearly conflict-free), L2 policies evict_first for the
// streaming x / X and evict_last for the Y ring, and the A task's 16
// four-step twiddles loaded into registers before its transform.
// ---------------------------------------------------------------------------
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

struct AbTmaCfg {
    static constexpr size_t STAGE = 16 * 256 * 8;   // dense 16 x 256 box
    static constexpr int LS = pad16c(256) + 1;      // engine line stride
    static constexpr size_t LINES = 16 * LS * 8;    // engine buffer, also the output staging (>= STAGE)
    static constexpr size_t LINES_OFF = 2 * STAGE;  // 1024-B aligned (the swizzled B staging)
    static constexpr size_t BAR_OFF = LINES_OFF + LINES;
    static constexpr size_t SMEM = BAR_OFF + 16;
};

template <bool INV>
__global__ void __launch_bounds__(256, 2)
    k_ab_tma(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yst,
             const __grid_constant__ CUtensorMap map_yld, const __grid_constant__ CUtensorMap map_out, int64_t batch,
             float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbBulkCtl ctl,
             const float2* /*ring: same signature as k_ab_ws*/, int /*opts*/) {
    using G = AbTmaCfg;
    using F = LineFFT<float, 256, 16, INV>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    float2* lines = reinterpret_cast<float2*>(smem_raw + G::LINES_OFF);
    const uint32_t lines_s = s_base + (uint32_t)G::LINES_OFF;
    const uint32_t bar0 = s_base + (uint32_t)G::BAR_OFF;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp), ntasks = 32 * batch;
    const uint64_t pol_stream = tmaops::policy_evict_first();
    const uint64_t pol_keep = tmaops::policy_evict_last();

    auto decode = [&](int64_t i, bool& isb, int64_t& b, int& part) {
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
    };
    // thread 0 only: task i's 16 x 256 input tile -> stage s
    auto issue = [&](int64_t i, int s) {
        if (i >= ntasks) return;
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
        const uint32_t bar = bar0 + 8 * s;
        if (!isb) {
            bk_arrive_expect(bar, (uint32_t)G::STAGE);
            tmaops::load3(st, &map_x, part * 16, 0, (int)b, bar, pol_stream);
        } else {
            while (bk_ld_acquire(ctl.done_a + b) < 16) __nanosleep(64);
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            bk_arrive_expect(bar, (uint32_t)G::STAGE);
            tmaops::load3(st, &map_yld, 0, part * 16, (int)(b % ctl.ring), bar, pol_keep);
        }
    };

    if (tid == 0) {
        bk_mbar_init(bar0, 1);
        bk_mbar_init(bar0 + 8, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        issue(blockIdx.x, 0);
        issue(blockIdx.x + gridDim.x, 1);
    }
    __syncthreads();

    int64_t prev_a = -1;
    for (int64_t k = 0;; ++k) {
        const int64_t i = blockIdx.x + k * gridDim.x;
        if (i >= ntasks) break;
        const int s = (int)(k & 1);
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        const int t = isb ? tid / 16 : tid % 16, l = isb ? tid % 16 : tid / 16;
        float2 w[16];
        if (!isb) {  // the A task's four-step twiddles W_N^{n1 k2}, k2 = l + 16 m
            const float2* tp = tw4 + (int64_t)l * 256 + part * 16 + t;
#pragma unroll
            for (int m = 0; m < 16; ++m) w[m] = __ldg(tp + (int64_t)m * 16 * 256);
        }
        if (tid == 0) bk_store_wait_all();  // previous task's store: staging free, Y (if A) complete
        bk_wait(bar0 + 8 * s, (uint32_t)((k >> 1) & 1));
        const float2* st = reinterpret_cast<const float2*>(smem_raw + s * G::STAGE);
        float2 v[16];
        if (!isb) {  // box [n2][16 n1]
#pragma unroll
            for (int m = 0; m < 16; ++m) v[F::pos_in(m)] = st[(l + 16 * m) * 16 + t];
        } else {  // box [16 k2][n1]
#pragma unroll
            for (int m = 0; m < 16; ++m) v[F::pos_in(m)] = st[t * 256 + l + 16 * m];
        }
        __syncthreads();  // stage s consumed, the staging is free
        if (tid == 0) {
            if (prev_a >= 0) {
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + prev_a, 1);
            }
            if (isb) bk_red_release(ctl.done_b + b, 1);
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            issue(i + 2 * gridDim.x, s);
        }
        prev_a = -1;
        F::run(v, lines + t * G::LS, l, tw256);
        __syncthreads();  // the line buffer becomes the output staging
        if (!isb) {  // Y box [k2][16 n1], dense
#pragma unroll
            for (int m = 0; m < 16; ++m) lines[(l + 16 * m) * 16 + t] = cmul_dir<INV>(v[F::pos_out(m)], w[m]);
        } else {  // X box [k1][16 k2] with the 128-B swizzle: chunk (k2 / 2) ^ (k1 % 8)
            char* sb = reinterpret_cast<char*>(lines);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int k1 = l + 16 * m;
                *reinterpret_cast<float2*>(sb + k1 * 128 + (((t >> 1) ^ (k1 & 7)) << 4) + ((t & 1) << 3)) =
                    cscale(v[F::pos_out(m)], scale);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (tid == 0) {
            if (!isb) {
                if (b >= ctl.ring)
                    while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(64);
                tmaops::store3(&map_yst, part * 16, 0, (int)(b % ctl.ring), lines_s, pol_keep);
                prev_a = b;
            } else {
                tmaops::store3(&map_out, part * 16, 0, (int)b, lines_s, pol_stream);
            }
        }
    }
    if (tid == 0) {
        bk_store_wait_all();
        if (prev_a >= 0) {
            asm volatile("fence.proxy.async.global;\n" ::: "memory");
            bk_red_release(ctl.done_a + prev_a, 1);
        }
    }
}

// ---------------------------------------------------------------------------
// Variant 42: warp-specialised form of 41.  8 compute warps + 1 producer
// warp per CTA, 2 CTAs/SM, a ring of NS = 3 smem stages of 32 KiB.  Each
// stage is used IN PLACE for its whole task: the TMA box lands in it, the
// engine exchanges inside it (A: the dense [256][16] column box, LineFFT
// LAYOUT 2; B: the 16 contiguous 2 KiB rows, XOR-swizzled LAYOUT 1), the
// results are written back into it as the output box (B with the 128-B TMA
// swizzle) and the producer stores it from there.  The producer alone
// issues loads (with the B dependency spin), stores, waits for their
// completion and signals done_a / done_b, so the compute warps only ever wait
// on the stage's full barrier and on their own named barrier.
// ---------------------------------------------------------------------------
template <int NS_ = 3>
struct AbWsCfgN {
    static constexpr int NS = NS_;
    static constexpr size_t STAGE = 16 * 256 * 8;
    static constexpr size_t BAR_OFF = NS * STAGE;  // full[NS], comp[NS]
    static constexpr size_t SMEM = BAR_OFF + 16 * NS;
};
using AbWsCfg = AbWsCfgN<3>;

template <bool INV, int NSV = 3>
__global__ void __launch_bounds__(288, NSV == 2 ? 3 : (NSV == 3 ? 2 : 1))
    k_ab_ws(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yst,
            const __grid_constant__ CUtensorMap map_yld, const __grid_constant__ CUtensorMap map_out, int64_t batch,
            float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbBulkCtl ctl,
            const float2* ring, int opts) {
    using G = AbWsCfgN<NSV>;
    constexpr int NS = G::NS;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, comp0 = full0 + 8 * NS;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp), ntasks = 32 * batch;

    auto decode = [&](int64_t i, bool& isb, int64_t& b, int& part) {
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
    };

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            bk_mbar_init(full0 + 8 * s, 1);
            bk_mbar_init(comp0 + 8 * s, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t my_tasks = ntasks > blockIdx.x ? (ntasks - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid >= 256) {  // ---- producer warp: lane 0 drives the TMA, all lanes discard ----
        const int lane = tid - 256;
        const bool l0 = lane == 0;
        // only lane 0 works unless the L2 discard of consumed Y rows is on
        const unsigned pmask = (opts & 1) ? 0xffffffffu : 1u;
        if (!((pmask >> lane) & 1u)) return;
        const uint64_t pol_stream = tmaops::policy_evict_first();
        const uint64_t pol_keep = tmaops::policy_evict_last();
        auto load = [&](int64_t k) {
            const int64_t i = blockIdx.x + k * gridDim.x;
            bool isb;
            int64_t b;
            int part;
            decode(i, isb, b, part);
            const int s = (int)(k % NS);
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
            if (!l0) return;
            if (!isb) {
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_x, part * 16, 0, (int)b, bar, pol_stream);
            } else {
                if (opts & 512) {
                    // timing experiment only (WRONG results): no A -> B dependency wait
                } else if (opts & 256) {
                    bk_wait_count(ctl.done_a + b, 16);
                } else {
                    while (bk_ld_acquire(ctl.done_a + b) < 16) __nanosleep(32);
                }
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_yld, 0, part * 16, (int)(b % ctl.ring), bar, (opts & 1024) ? pol_stream : pol_keep);
            }
        };
        int64_t pend_a = -1;  // transform whose A store is the newest bulk group, signalled once complete
        auto store = [&](int64_t k) {  // task k's outputs are in its stage
            const int64_t i = blockIdx.x + k * gridDim.x;
            bool isb;
            int64_t b;
            int part;
            decode(i, isb, b, part);
            const int s = (int)(k % NS);
            bk_wait(comp0 + 8 * s, (uint32_t)((k / NS) & 1));
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
            const bool discard = (opts & 1) != 0, defer = (opts & 2) != 0;
            if (isb && discard) {
                // its Y rows were read (loaded) before its compute: drop the
                // dead lines from L2 without write-back (256 lines of 128 B)
                const float2* y = ring + (b % ctl.ring) * 65536 + (int64_t)part * 16 * 256;
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(y + (lane + 32 * q) * 16) : "memory");
                __syncwarp(pmask);
            }
            if (l0) {
                if (!isb) {
                    if (b >= ctl.ring && !(opts & 512)) {
                        if (opts & 256)
                            bk_wait_count(ctl.done_b + (b - ctl.ring), 16);
                        else
                            while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(32);
                    }
                    tmaops::store3(&map_yst, part * 16, 0, (int)(b % ctl.ring), st, pol_keep);
                } else {
                    bk_red_release(ctl.done_b + b, 1);  // the ring slot rows are free
                    tmaops::store3(&map_out, part * 16, 0, (int)b, st, pol_stream);
                }
                if (defer) {
                    // every group but this newest one is complete: signal the previous A
                    asm volatile("cp.async.bulk.wait_group 1;\n" ::: "memory");
                    if (pend_a >= 0) {
                        asm volatile("fence.proxy.async.global;\n" ::: "memory");
                        bk_red_release(ctl.done_a + pend_a, 1);
                    }
                    pend_a = isb ? -1 : b;
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // stage reusable
                } else if (!isb && (opts & 8)) {
                    // stage reusable once read; the completion wait and the
                    // signal follow right after the next load is issued
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
                    pend_a = b;
                } else if (!isb) {
                    bk_store_wait_all();  // Y rows written: signal now (B tasks of other CTAs wait on it)
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");
                    bk_red_release(ctl.done_a + b, 1);
                } else {
                    asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // stage reusable
                }
            }
            __syncwarp(pmask);
        };
        const int pf = (opts >> 4) & 7;  // L2 prefetch distance (tasks) for A tiles, 0 = off
        for (int64_t k = 0; k < my_tasks; ++k) {
            if (k >= NS) store(k - NS);
            load(k);
            if (pf && l0 && k + pf < my_tasks) {  // warm L2 with a later A task's HBM tile
                bool pb;
                int64_t pbb;
                int ppart;
                decode(blockIdx.x + (k + pf) * gridDim.x, pb, pbb, ppart);
                if (!pb) tmaops::prefetch3(&map_x, ppart * 16, 0, (int)pbb);
            }
            if ((opts & 8) && l0 && pend_a >= 0) {
                bk_store_wait_all();
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + pend_a, 1);
                pend_a = -1;
            }
            __syncwarp(pmask);
        }
        for (int64_t k = (my_tasks > NS ? my_tasks - NS : 0); k < my_tasks; ++k) store(k);
        if (l0) {
            bk_store_wait_all();
            if (pend_a >= 0) {
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + pend_a, 1);
            }
        }
        return;
    }

    // ---- compute warps (256 threads) ----
#ifndef B200FFT_AB_TWREC
#define B200FFT_AB_TWREC 1
#endif
    using FA = LineFFT<float, 256, 16, INV, 2, false, (B200FFT_AB_TWREC != 0)>;
    using FB = LineFFT<float, 256, 16, INV, 1, false, (B200FFT_AB_TWREC != 0)>;
    for (int64_t k = 0; k < my_tasks; ++k) {
        const int64_t i = blockIdx.x + k * gridDim.x;
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        float2 v[16];
        if (!isb) {
            const int t = tid % 16, l = tid / 16;  // line = column n1 = 16 part + t
            const float2* tp = tw4 + (int64_t)l * 256 + part * 16 + t;
            // the four-step twiddles: prefetched before the stage wait when
            // registers allow (3 stages, 2 CTAs/SM), else loaded at use
            constexpr int NPF = NSV >= 3 ? 16 : 1;
            float2 w[NPF];
            if constexpr (NPF == 16) {
#pragma unroll
                for (int m = 0; m < 16; ++m) w[m] = __ldg(tp + (int64_t)m * 16 * 256);
            }
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FA::pos_in(m)] = line[FA::bpos(l, m)];
            FA::run(v, line, l, tw256, -256);
            FA::lsync(-256);
            if (NPF == 16 || !(opts & 128)) {
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    const float2 wm = (NPF == 16) ? w[m % NPF] : __ldg(tp + (int64_t)m * 16 * 256);
                    line[(l + 16 * m) * 16] = cmul_dir<INV>(v[FA::pos_out(m)], wm);
                }
            } else {
                // W_N^{n1 (l + 16 m)} = W_N^{n1 l} (W_N^{16 n1})^m: two table
                // entries and a 15-step product (fp32, ~15 ulp) instead of 16 loads
                float2 wm = __ldg(tp);
                const float2 ws = __ldg(tw4 + (int64_t)16 * 256 + part * 16 + t);
#pragma unroll
                for (int m = 0; m < 16; ++m) {
                    line[(l + 16 * m) * 16] = cmul_dir<INV>(v[FA::pos_out(m)], wm);
                    wm = cmul(wm, ws);
                }
            }
        } else {
            const int t = tid / 16, l = tid % 16;  // line = row k2 = 16 part + t of Y
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            if (opts & 4) {  // the Y rows are in smem now: drop their 256 L2 lines (one per thread)
                const float2* y = ring + (b % ctl.ring) * 65536 + (int64_t)part * 16 * 256 + tid * 16;
                asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(y) : "memory");
            }
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

// ---------------------------------------------------------------------------
// Variants 45 / 46: k_ab_ws with 8-line tasks (16 KiB stages, 32 A + 32 B
// parts per transform).  The same 8 compute warps per CTA run ONE task at a
// time with E = 8 (steps 8, 8, 4): A with the 8 columns as the thread-fastest
// index (LineFFT LAYOUT 4, conflict-free in the dense [256][8] box), B with
// one warp per row (LAYOUT 3, warp-synchronous exchanges).  Half the stage
// size at the same stage memory per SM means NS - 1 of NS stages can be in
// flight instead of 1 of 2: 45 = 3 CTAs/SM x 4 stages, 46 = 4 CTAs/SM x 3.
// ---------------------------------------------------------------------------
template <int NS_>
struct AbWs8Cfg {
    static constexpr int NS = NS_;
    static constexpr size_t STAGE = 8 * 256 * 8;
    static constexpr size_t BAR_OFF = NS * STAGE;
    static constexpr size_t SMEM = BAR_OFF + 16 * NS;
};

template <bool INV, int NS, int MINB>
__global__ void __launch_bounds__(288, MINB)
    k_ab_ws8(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yst,
             const __grid_constant__ CUtensorMap map_yld, const __grid_constant__ CUtensorMap map_out, int64_t batch,
             float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbBulkCtl ctl,
             const float2* ring, int opts) {
    using G = AbWs8Cfg<NS>;
    constexpr int PP = 32;  // parts per phase
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, comp0 = full0 + 8 * NS;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = PP * Dp, n2t = 2 * PP * (batch - Dp), ntasks = 2 * PP * batch;
    (void)ring;

    auto decode = [&](int64_t i, bool& isb, int64_t& b, int& part) {
        if (i < n1t) {
            isb = false;
            b = i / PP;
            part = (int)(i % PP);
        } else if (i < n1t + n2t) {
            const int64_t j = i - n1t, r = j % (2 * PP);
            isb = r >= PP;
            b = Dp + j / (2 * PP) - (isb ? Dp : 0);
            part = (int)(r % PP);
        } else {
            const int64_t j = i - n1t - n2t;
            isb = true;
            b = batch - Dp + j / PP;
            part = (int)(j % PP);
        }
    };

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
            decode(blockIdx.x + k * gridDim.x, isb, b, part);
            const int s = (int)(k % NS);
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
            if (!isb) {
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_x, part * 8, 0, (int)b, bar, pol_stream);
            } else {
                while (bk_ld_acquire(ctl.done_a + b) < PP) __nanosleep(32);
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_yld, 0, part * 8, (int)(b % ctl.ring), bar, pol_keep);
            }
        };
        auto store = [&](int64_t k) {
            bool isb;
            int64_t b;
            int part;
            decode(blockIdx.x + k * gridDim.x, isb, b, part);
            const int s = (int)(k % NS);
            bk_wait(comp0 + 8 * s, (uint32_t)((k / NS) & 1));
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
            if (!isb) {
                if (b >= ctl.ring)
                    while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < PP) __nanosleep(32);
                tmaops::store3(&map_yst, part * 8, 0, (int)(b % ctl.ring), st, pol_keep);
                bk_store_wait_all();  // Y rows written: B tasks of other CTAs wait on the signal
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_red_release(ctl.done_a + b, 1);
            } else {
                bk_red_release(ctl.done_b + b, 1);  // its ring rows were read at load
                tmaops::store3(&map_out, part * 8, 0, (int)b, st, pol_stream);
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // stage reusable
            }
        };
        const int pf = (opts >> 4) & 7;
        for (int64_t k = 0; k < my_tasks; ++k) {
            if (k >= NS) store(k - NS);
            load(k);
            if (pf && k + pf < my_tasks) {
                bool pb;
                int64_t pbb;
                int ppart;
                decode(blockIdx.x + (k + pf) * gridDim.x, pb, pbb, ppart);
                if (!pb) tmaops::prefetch3(&map_x, ppart * 8, 0, (int)pbb);
            }
        }
        for (int64_t k = (my_tasks > NS ? my_tasks - NS : 0); k < my_tasks; ++k) store(k);
        bk_store_wait_all();
        return;
    }

    // ---- compute warps (256 threads, one task at a time) ----
    using FA = LineFFT<float, 256, 8, INV, 4, false, true>;
    using FB = LineFFT<float, 256, 8, INV, 3, false, true>;
    for (int64_t k = 0; k < my_tasks; ++k) {
        bool isb;
        int64_t b;
        int part;
        decode(blockIdx.x + k * gridDim.x, isb, b, part);
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        float2 v[8];
        if (!isb) {
            const int t = tid & 7, l = tid >> 3;  // line = column n1 = 8 part + t
            const int n1 = part * 8 + t;
            float2 wm = __ldg(tw4 + (int64_t)l * 256 + n1);    // W_N^{n1 l}
            const float2 ws = __ldg(tw4 + (int64_t)32 * 256 + n1);  // W_N^{32 n1}
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t;
#pragma unroll
            for (int m = 0; m < 8; ++m) v[FA::pos_in(m)] = line[(l + 32 * m) * 8];  // dense, as landed
            FA::run(v, line, l, tw256, -256);
            FA::lsync(-256);
#pragma unroll
            for (int m = 0; m < 8; ++m) {  // Y[k2 = l + 32 m][n1] * W_N^{n1 k2}, dense for the store
                line[(l + 32 * m) * 8] = cmul_dir<INV>(v[FA::pos_out(m)], wm);
                wm = cmul(wm, ws);
            }
        } else {
            const int t = tid >> 5, l = tid & 31;  // line = row k2 = 8 part + t of Y (one warp)
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t * 256;
#pragma unroll
            for (int m = 0; m < 8; ++m) v[FB::pos_in(m)] = line[l + 32 * m];  // as landed
            FB::run(v, line, l, tw256, -32);
            FB::lsync(-256);  // the output box spans every warp's row
            char* sb = reinterpret_cast<char*>(st);  // X box [k1][8 k2], 64-B TMA swizzle
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int k1 = l + 32 * m;
                *reinterpret_cast<float2*>(sb + k1 * 64 + (((t >> 1) ^ ((k1 >> 1) & 3)) << 4) + ((t & 1) << 3)) =
                    cscale(v[FB::pos_out(m)], scale);
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        bk_arrive(comp0 + 8 * s);
    }
}

// ---------------------------------------------------------------------------
// Variant 47: k_ab_ws (44) with the A tasks' Y rows stored by the compute
// warps straight from registers (coalesced 128-B rows: the 16 columns of a
// task are the thread-fastest index), so an A task's stage is free as soon
// as its last exchange has been read -- the producer reloads it while the
// compute warps are still storing.  Publication: every compute thread
// fences its stores (fence.acq_rel.gpu) and arrives on the stage's pub
// barrier; the producer waits for it after issuing the next load, then
// releases done_a.  The ring-slot check moves from the A store to the A
// load.  B tasks are unchanged (TMA box store).
// ---------------------------------------------------------------------------
struct AbDsCfg {
    static constexpr int NS = 2;
    static constexpr size_t STAGE = 16 * 256 * 8;
    static constexpr size_t BAR_OFF = NS * STAGE;  // full[NS], comp[NS], pub[NS]
    static constexpr size_t SMEM = BAR_OFF + 24 * NS;
};

template <bool INV>
__global__ void __launch_bounds__(288, 3)
    k_ab_ds(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yst,
            const __grid_constant__ CUtensorMap map_yld, const __grid_constant__ CUtensorMap map_out, int64_t batch,
            float scale, const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbBulkCtl ctl,
            const float2* ring, int opts) {
    using G = AbDsCfg;
    constexpr int NS = G::NS;
    (void)map_yst;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, comp0 = full0 + 8 * NS, pub0 = comp0 + 8 * NS;
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp), ntasks = 32 * batch;

    auto decode = [&](int64_t i, bool& isb, int64_t& b, int& part) {
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
    };

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            bk_mbar_init(full0 + 8 * s, 1);
            bk_mbar_init(comp0 + 8 * s, 256);
            bk_mbar_init(pub0 + 8 * s, 256);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    const int64_t my_tasks = ntasks > blockIdx.x ? (ntasks - 1 - blockIdx.x) / gridDim.x + 1 : 0;

    if (tid >= 256) {  // ---- producer: lane 0 ----
        if (tid != 256) return;
        const uint64_t pol_stream = tmaops::policy_evict_first();
        const uint64_t pol_keep = tmaops::policy_evict_last();
        int npub[NS] = {};  // A tasks published per stage so far (pub barrier phases)
        auto load = [&](int64_t k) {
            bool isb;
            int64_t b;
            int part;
            decode(blockIdx.x + k * gridDim.x, isb, b, part);
            const int s = (int)(k % NS);
            const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
            if (!isb) {
                // the compute warps will store this task's Y rows into the ring slot
                if (b >= ctl.ring)
                    while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(32);
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_x, part * 16, 0, (int)b, bar, pol_stream);
            } else {
                while (bk_ld_acquire(ctl.done_a + b) < 16) __nanosleep(32);
                asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                tmaops::load3(st, &map_yld, 0, part * 16, (int)(b % ctl.ring), bar, pol_keep);
            }
        };
        // stage of task k free (A: its exchanges read; B: its X box stored)
        auto finish = [&](int64_t k) {
            bool isb;
            int64_t b;
            int part;
            decode(blockIdx.x + k * gridDim.x, isb, b, part);
            const int s = (int)(k % NS);
            bk_wait(comp0 + 8 * s, (uint32_t)((k / NS) & 1));
            if (isb) {
                const uint32_t st = s_base + (uint32_t)(s * G::STAGE);
                bk_red_release(ctl.done_b + b, 1);  // its ring rows were read at load
                tmaops::store3(&map_out, part * 16, 0, (int)b, st, pol_stream);
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            }
        };
        // task k's Y rows globally visible: release done_a
        auto publish = [&](int64_t k) {
            bool isb;
            int64_t b;
            int part;
            decode(blockIdx.x + k * gridDim.x, isb, b, part);
            if (isb) return;
            const int s = (int)(k % NS);
            bk_wait(pub0 + 8 * s, (uint32_t)(npub[s] & 1));
            ++npub[s];
            bk_red_release(ctl.done_a + b, 1);
        };
        const int pf = (opts >> 4) & 7;
        for (int64_t k = 0; k < my_tasks; ++k) {
            if (k >= NS) finish(k - NS);
            load(k);
            if (k >= NS) publish(k - NS);
            if (pf && k + pf < my_tasks) {
                bool pb;
                int64_t pbb;
                int ppart;
                decode(blockIdx.x + (k + pf) * gridDim.x, pb, pbb, ppart);
                if (!pb) tmaops::prefetch3(&map_x, ppart * 16, 0, (int)pbb);
            }
        }
        for (int64_t k = (my_tasks > NS ? my_tasks - NS : 0); k < my_tasks; ++k) {
            finish(k);
            publish(k);
        }
        bk_store_wait_all();
        return;
    }

    // ---- compute warps (256 threads) ----
    using FA = LineFFT<float, 256, 16, INV, 2, false, true>;
    using FB = LineFFT<float, 256, 16, INV, 1, false, true>;
    float2* yring = const_cast<float2*>(ring);
    for (int64_t k = 0; k < my_tasks; ++k) {
        bool isb;
        int64_t b;
        int part;
        decode(blockIdx.x + k * gridDim.x, isb, b, part);
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
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            bk_arrive(comp0 + 8 * s);  // this thread is done with the stage
            float2 wm = __ldg(tp);
            const float2 ws = __ldg(tw4 + (int64_t)16 * 256 + part * 16 + t);
            float2* y = yring + (b % ctl.ring) * 65536 + part * 16 + t;
#pragma unroll
            for (int m = 0; m < 16; ++m) {  // Y[k2 = l + 16 m][n1]: 16 threads = one 128-B row segment
                y[(l + 16 * m) * 256] = cmul_dir<INV>(v[FA::pos_out(m)], wm);
                wm = cmul(wm, ws);
            }
            asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
            bk_arrive(pub0 + 8 * s);
        } else {
            const int t = tid / 16, l = tid % 16;  // line = row k2 = 16 part + t of Y
            bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
            float2* line = st + t * 256;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FB::pos_in(m)] = line[l + 16 * m];
            FB::run(v, line, l, tw256, -256);
            FB::lsync(-256);
            char* sb = reinterpret_cast<char*>(st);
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                const int k1 = l + 16 * m;
                *reinterpret_cast<float2*>(sb + k1 * 128 + (((t >> 1) ^ (k1 & 7)) << 4) + ((t & 1) << 3)) =
                    cscale(v[FB::pos_out(m)], scale);
            }
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            bk_arrive(comp0 + 8 * s);
        }
    }
}

}  // namespace b200fft
