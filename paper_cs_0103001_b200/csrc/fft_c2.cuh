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
    int* done_a;                    // [batch] A parts of transform b whose Y rows are in the ring
    int* done_b;                    // [batch] B parts of transform b that have read their Y rows
    unsigned long long* next;       // next task position to take (k_ab_st)
    int D, ring;                    // dependency distance (transforms), ring slots
};

// optional outer four-step twiddle fused into the 32768-point B epilogue
// (the distributed 2^30 four-step's step (T), else k_twiddle4): output k of
// transform b times W_n^{(row0 + b) k}, W_n^x = a[x >> sh] * b[x & mask]
// (fp64-generated tables, x < n: no wrap); a == nullptr: none
struct OuterTw {
    const float2* a;
    const float2* b;
    int sh;
    int64_t row0;
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
// wait for the phase with the given parity; the try_wait carries a suspend
// time hint, so a waiting thread sleeps until the phase completes (or the
// hint expires) instead of spinning -- spinning waits had been a third of
// the executed instructions of the task pipelines (ncu), issue slots taken
// from the compute warps
__device__ __forceinline__ void bk_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "BK_WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra BK_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(20000u)
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

// position i of the global task order -> (is B, transform b, part p), T A
// tasks and T B tasks per transform (T = 16 for N = 65536, 8 for 32768)
template <int T = 16>
__device__ __forceinline__ void ab_decode(int64_t i, int64_t batch, int64_t Dp, bool& isb, int64_t& b, int& part) {
    const int64_t n1t = T * Dp, n2t = 2 * T * (batch - Dp);
    if (i < n1t) {
        isb = false;
        b = i / T;
        part = (int)(i % T);
    } else if (i < n1t + n2t) {
        const int64_t j = i - n1t, r = j % (2 * T);
        isb = r >= T;
        b = Dp + j / (2 * T) - (isb ? Dp : 0);
        part = (int)(r % T);
    } else {
        const int64_t j = i - n1t - n2t;
        isb = true;
        b = batch - Dp + j / T;
        part = (int)(j % T);
    }
}

// XOR layout of a 32-line x 128-point exchange (element x of line L at
// x * 32 + (L ^ 2 ((x / 16) mod 8))): conflict-free for the 8-lanes-per-line
// writes and the line-fastest reads (k_big pass 2, st_task_b128)
__device__ __forceinline__ int big_bx(int x, int line) { return x * 32 + (line ^ (((x >> 4) & 7) << 1)); }

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


// ---------------------------------------------------------------------------
// k_ab_st: the same tasks, with the outputs stored straight from registers
// and the tasks handed out dynamically.  Per CTA: 8 compute warps, a
// producer (warp 8, lane 0), a signaller (warp 9, lane 0); NS stages of
// 32 KiB.  A stage holds its task only from the TMA load until the compute
// warps have read their step-1 inputs: the step-0 results are exchanged IN
// the stage (after a compute-group barrier), then the stage is released
// (mbarrier "empty") and the producer refills it while step 1, the twiddles
// and the stores run from registers -- no output staging, no store
// completion holding a stage, 32 B of smem traffic per element and task.
//   A(b, p): thread (t, l) = (tid % 16, tid / 16) holds column n1 = 16p + t,
//            elements n2 = l + 16 r (the dense [256 n2][16 n1] box); step 0
//            (radix 16) -> exchange (element x of line t at x * 16 + t) ->
//            step 1 -> k2 = l + 16 q; Y[k2][n1] = . * W_N^{n1 k2} * scale
//            stored as 128-B row segments (16 adjacent t).
//   B(b, p): step 0 with (line r, lane l') = (tid / 16, tid % 16) on the 16
//            dense Y rows k2 = 16p + r; exchange in the XOR layout x * 16 +
//            (line ^ (x / 16 mod 16)), conflict-free for both mappings; step
//            1 with (line t, lane l) = (tid % 16, tid / 16): k1 = l + 16 q;
//            X[k2 + 256 k1] stored as 128-B segments (16 adjacent k2).
// The scale (the paper's 1/N, a power of two: exact) is folded
// into the A twiddle, i.e. applied to Y: bit-identical to scaling X.
// Signals: after an A task's Y stores every compute thread arrives on a
// signal mbarrier (release, CTA scope); the signaller waits on it (acquire),
// makes the stores visible at gpu scope (fence.acq_rel.gpu, cumulative) and
// counts the task in done_a -- one fence per task, off the compute warps.
// Scheduling: the producer takes the next position of the global task order
// from an atomic counter (no static round robin: CTAs that run slower take
// fewer tasks, so no transform's B parts wait on a straggler's A part).
// Deadlock freedom: every wait (a B load on done_a, an A load on its ring
// slot's done_b, a signal slot) points at tasks taken earlier, and no signal
// waits for a later load; all CTAs are co-resident (cooperative launch).
// ---------------------------------------------------------------------------
template <int NS_>
struct AbStCfg {
    static constexpr int NS = NS_;
    static constexpr int NSIG = 4;  // A tasks a CTA may have computed but not yet signalled
    static constexpr size_t STAGE = 16 * 256 * 8;
    static constexpr size_t BAR_OFF = NS * STAGE;                       // full[NS], empty[NS], sig[NSIG]
    static constexpr size_t INFO_OFF = BAR_OFF + 8 * (2 * NS + NSIG);   // task[NS], sigb[NSIG] (int64), sigdone
    static constexpr size_t SMEM = INFO_OFF + 8 * (NS + NSIG) + 16;
};

// step-1 twiddles W_256^{l r} from the constant table (fft_engine.cuh
// c_w256): a thread's depend only on its lane l, two distinct l per warp
template <bool INV>
__device__ __forceinline__ void st_step1_twiddle_c(float2* v, int l) {
#pragma unroll
    for (int r = 1; r < 16; ++r) v[r] = cmul_dir<INV>(v[r], c_w256[(l * r) & 255]);
}

template <bool INV>
__device__ __forceinline__ void st_step1_twiddle(float2* v, int l, const float2* __restrict__ tw256) {
    // step 1 of the 256-point Stockham (span 16): v[r] *= W_256^{l r}, r < 16,
    // as powers of the one step-major table entry W_256^l (fp32, ~15 ulp;
    // loading the 15 entries instead measured 1% slower, a four-chain product
    // 0.6% slower)
    const float2 w1 = __ldg(tw256 + tw_off(256, 1, 4) + l);
    float2 w = w1;
#pragma unroll
    for (int r = 1; r < 16; ++r) {
        v[r] = cmul_dir<INV>(v[r], w);
        if (r < 15) w = cmul(w, w1);
    }
}

// ---------------------------------------------------------------------------
// The two task bodies of k_ab_st, for one compute group of 256 threads (lo, hi) = (tid % 16,
// tid / 16) on the stage st; `bar` is the group's named barrier.  Each
// releases the stage (arrive on `empty`) as soon as its step-1 inputs are in
// registers.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void grp_sync(int bar) { asm volatile("bar.sync %0, 256;\n" ::"r"(bar) : "memory"); }

// 8-byte global store with an L2 eviction-priority policy (createpolicy)
__device__ __forceinline__ void st_pol(float2* p, float2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;\n" ::"l"(p), "f"(v.x), "f"(v.y), "l"(pol)
                 : "memory");
}

template <bool INV, int N1 = 256>
__device__ __forceinline__ void st_task_a(float2* st, int lo, int hi, int bar, uint32_t empty, int part, float2* y0,
                                          float scale, const float2* __restrict__ tw4,
                                          const float2* __restrict__ tw256, int xo) {
    // the four-step twiddle's two table entries, loaded before the FFT so
    // their latency hides behind it (after the exchange: 1.3% slower, round 2)
    const int n1 = part * 16 + lo;
    const float2 wm0 = __ldg(tw4 + (int64_t)hi * N1 + n1);
    const float2 ws = __ldg(tw4 + (int64_t)16 * N1 + n1);
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = st[(hi + 16 * r) * 16 + lo];
    if (!(xo & 8)) dft<16, INV>(v);
    if (!(xo & 64)) {
        grp_sync(bar);
#pragma unroll
        for (int q = 0; q < 16; ++q) st[(16 * hi + q) * 16 + lo] = v[q];
        grp_sync(bar);
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = st[(hi + 16 * r) * 16 + lo];
    }
    bk_arrive(empty);
    if (!(xo & 8)) {
        if (xo & 4096) st_step1_twiddle<INV>(v, hi, tw256);  // the round-2 recurrence (3% slower)
        else st_step1_twiddle_c<INV>(v, hi);
        dft<16, INV>(v);
    }
    // Y[k2][n1] = v[q] * W_N^{n1 k2} * scale, k2 = hi + 16 q
    float2 wm = cscale(wm0, scale);
    // N1 = 128: Y rows stored with column n1 ^ 8 (k2 mod 4) (k2 mod 4 = hi mod
    // 4 here) so that st_task_b128's step-0 reads of 4 rows per warp hit
    // distinct banks (1 KiB rows alone put them on the same 16 banks)
    const int yc = N1 == 128 ? (n1 ^ (8 * (hi & 3))) : n1;
    float2* y = y0 + (int64_t)hi * N1 + yc;
    const uint64_t keep = tmaops::policy_evict_last();
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        // Y without a cache hint (the ring is persisting by the launch's
        // access-policy window): evict-last stores measured 1.3% slower
        // (xo 16384 selects them, for comparisons)
        if (xo & 16384) {
            if (!(xo & 2) || v[q].x == 1.2345e-38f) st_pol(y + q * 16 * N1, cmul_dir<INV>(v[q], wm), keep);
        } else if (!(xo & 2) || v[q].x == 1.2345e-38f) y[q * 16 * N1] = cmul_dir<INV>(v[q], wm);
        if (q < 15) wm = cmul(wm, ws);
    }
}

template <bool INV>
__device__ __forceinline__ void st_task_b(float2* st, int lo, int hi, int bar, uint32_t empty, float2* x0,
                                          const float2* __restrict__ tw256, int xo) {
    float2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = st[hi * 256 + lo + 16 * r];
    if (!(xo & 8)) dft<16, INV>(v);
    if (!(xo & 64)) {
        grp_sync(bar);
#pragma unroll
        for (int q = 0; q < 16; ++q) st[(16 * lo + q) * 16 + (hi ^ lo)] = v[q];
        grp_sync(bar);
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = st[(hi + 16 * r) * 16 + (lo ^ r)];
    }
    bk_arrive(empty);
    if (!(xo & 8)) {
        if (xo & 4096) st_step1_twiddle<INV>(v, hi, tw256);  // the round-2 recurrence (3% slower)
        else st_step1_twiddle_c<INV>(v, hi);
        dft<16, INV>(v);
    }
    float2* x = x0 + lo + (int64_t)hi * 256;
    // X is stored without a cache hint: evict-first stores measured 0.7-0.9%
    // slower (profiles/README.md, round 2 C2 experiments); xo bits 256 / 1024
    // select the .cs / evict-first / evict-last forms for timing comparisons
    const uint64_t stream = (xo & 1024) ? tmaops::policy_evict_last() : tmaops::policy_evict_first();
    if (xo & 2048) {  // timing experiment: each task writes one contiguous 32 KiB block (wrong order)
        float2* xc = x0 - (x0 - (float2*)nullptr) % 65536 + ((x0 - (float2*)nullptr) % 256) / 16 * 4096 + hi * 16 + lo;
#pragma unroll
        for (int q = 0; q < 16; ++q) st_pol(xc + q * 256, v[q], stream);
    } else if (xo & 256) {
#pragma unroll
        for (int q = 0; q < 16; ++q) __stcs(x + q * 16 * 256, v[q]);
    } else if (xo & (2 | 1024 | 128)) {
#pragma unroll
        for (int q = 0; q < 16; ++q)
            if (!(xo & 2) || v[q].x == 1.2345e-38f) st_pol(x + q * 16 * 256, v[q], stream);
    } else {
#pragma unroll
        for (int q = 0; q < 16; ++q) x[q * 16 * 256] = v[q];
    }
}

// B task body for N = 32768 (N1 = 128): the stage holds 32 Y rows k2 =
// 32 p + line of 128 points (as landed); 128-point DFTs over n1 = j + 8 r:
// step 0 radix 16 over r (8 lanes j per line), the XOR-layout exchange,
// step 1 radix 8 over j with W_128^{q j} (q = lt + 8 b, line-fastest):
// X[k2 + 256 k1], k1 = q + 16 m -- a warp stores 32 consecutive k2 (256 B).
template <bool INV, bool OTW>
__device__ __forceinline__ void st_task_b128(float2* st, int tid, int bar, uint32_t empty, float2* x0, OuterTw ow,
                                             int64_t tb, int k2base) {
    const int L0 = tid >> 3, j = tid & 7, sw = L0 & 3;  // row L0 stored with column ^ 8 (L0 mod 4)
    float2 v[16];
    const float2* src = st + L0 * 128 + j;
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = src[8 * (r ^ sw)];
    dft<16, INV>(v);
    grp_sync(bar);
#pragma unroll
    for (int q = 0; q < 16; ++q) st[big_bx(16 * j + q, L0)] = v[q];
    grp_sync(bar);
    const int line = tid & 31, lt = tid >> 5;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int q = lt + 8 * b;
#pragma unroll
        for (int r = 0; r < 8; ++r) v[b * 8 + r] = st[big_bx(q + 16 * r, line)];
    }
    bk_arrive(empty);
    // outer twiddle W^{R k}, k = k2 + 256 (q + 16 m): per b the value at m = 0
    // and the step W^{4096 R} (loaded here: their latency overlaps step 1)
    float2 ha[2], la[2], hs = make_float2(0.f, 0.f), ls = hs;
    const int64_t R = ow.row0 + tb, msk = ((int64_t)1 << ow.sh) - 1;
    if constexpr (OTW) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int64_t x = R * (int64_t)(k2base + line + 256 * (lt + 8 * b));
            ha[b] = __ldg(ow.a + (x >> ow.sh));
            la[b] = __ldg(ow.b + (x & msk));
        }
        const int64_t xs = R * 4096;
        hs = __ldg(ow.a + (xs >> ow.sh));
        ls = __ldg(ow.b + (xs & msk));
    }
#pragma unroll
    for (int b = 0; b < 2; ++b) {
        const int q = lt + 8 * b;
#pragma unroll
        for (int r = 1; r < 8; ++r) v[b * 8 + r] = cmul_dir<INV>(v[b * 8 + r], c_w256[(2 * q * r) & 255]);
        dft<8, INV>(v + b * 8);
    }
    if constexpr (OTW) {
        const float2 ws = cmul(hs, ls);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            float2 w = cmul(ha[b], la[b]);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                v[b * 8 + m] = cmul_dir<INV>(v[b * 8 + m], w);
                if (m < 7) w = cmul(w, ws);
            }
        }
    }
    float2* x = x0 + line;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int m = 0; m < 8; ++m) x[(int64_t)256 * (lt + 8 * b + 16 * m)] = v[b * 8 + m];
}

// L = 65536 (C2: N1 = N2 = 256, 16 A + 16 B tasks per transform) or 32768
// (N1 = 128, N2 = 256: 8 A tasks of 16 columns, 8 B tasks of 32 Y rows;
// OTW: with the outer four-step twiddle `ow` in the B epilogue)
template <bool INV, int NS, int MINB, int L = 65536, bool OTW = false>
__global__ void __launch_bounds__(320, MINB)
    k_ab_st(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_yld,
            float2* __restrict__ ring, float2* __restrict__ out, int64_t batch, float scale,
            const float2* __restrict__ tw4, const float2* __restrict__ tw256, AbCtl ctl, int opts, OuterTw ow) {
    using G = AbStCfg<NS>;
    constexpr int N1 = L / 256, T = N1 / 16, ROWS = 4096 / N1;  // B task: ROWS Y rows of N1
    constexpr int NSIG = G::NSIG;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, empty0 = full0 + 8 * NS, sig0 = empty0 + 8 * NS;
    volatile int64_t* task = reinterpret_cast<volatile int64_t*>(smem_raw + G::INFO_OFF);
    volatile int64_t* sigb = task + NS;
    volatile int* sigdone = reinterpret_cast<volatile int*>(sigb + NSIG);
    const int tid = threadIdx.x;
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t ntasks = 2 * T * batch;

    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            bk_mbar_init(full0 + 8 * s, 1);
            bk_mbar_init(empty0 + 8 * s, 256);
        }
        for (int j = 0; j < NSIG; ++j) bk_mbar_init(sig0 + 8 * j, 256);
        *sigdone = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    if (tid >= 256) {
        const int lane = tid & 31;
        if (lane != 0) return;
        if (tid < 288) {  // ---- producer ----
            const uint64_t pol_stream = (opts & 512) ? tmaops::policy_evict_last() : tmaops::policy_evict_first();
            const uint64_t pol_keep = tmaops::policy_evict_last();
            int na = 0;  // A tasks issued by this CTA
            // (taking the next position before the stage is free, relaxed
            // flag polling and L2 prefetches of later A boxes measured +4%,
            // +-0 and +1.5%: profiles/README.md)
            int64_t ipair = 0;
            for (int64_t k = 0;; ++k) {
                const int s = (int)(k % NS);
                if (k >= NS) bk_wait(empty0 + 8 * s, (uint32_t)(((k / NS) - 1) & 1));
                int64_t i;
                if (opts & 16) {
                    i = blockIdx.x + k * gridDim.x;
                } else if (opts & 32) {
                    if ((k & 1) == 0) ipair = (int64_t)atomicAdd(ctl.next, 2ull);
                    i = ipair + (k & 1);
                } else {
                    i = (int64_t)atomicAdd(ctl.next, 1ull);
                }
                task[s] = i;
                const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
                if (i >= ntasks) {  // no more work: the compute warps exit on this stage
                    bk_arrive(bar);
                    break;
                }
                bool isb;
                int64_t b;
                int part;
                ab_decode<T>(i, batch, Dp, isb, b, part);
                if (opts & 1) {  // timing experiment: no loads, no dependency waits
                    if (!isb) {
                        while (*sigdone < na - NSIG + 1) __nanosleep(20);
                        ++na;
                    }
                    bk_arrive(bar);
                } else if (!isb) {
                    // a free signal slot for this A task (the signaller is at most
                    // NSIG A tasks behind the compute warps)
                    while (*sigdone < na - NSIG + 1) __nanosleep(20);
                    ++na;
                    // the ring slot's previous transform: all its B parts have read it
                    if (b >= ctl.ring && !(opts & 4))
                        while (bk_ld_acquire(ctl.done_b + (b - ctl.ring)) < T) __nanosleep(32);
                    bk_arrive_expect(bar, (uint32_t)G::STAGE);
                    tmaops::load3(st, &map_x, part * 16, 0, (int)b, bar, pol_stream);
                } else {
                    if (!(opts & 4))
                        while (bk_ld_acquire(ctl.done_a + b) < T) __nanosleep(32);
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");
                    bk_arrive_expect(bar, (uint32_t)G::STAGE);
                    tmaops::load3(st, &map_yld, 0, part * ROWS, (int)(b % ctl.ring), bar, pol_keep);
                }
            }
        } else {  // ---- signaller ----
            for (int j = 0;; ++j) {
                bk_wait(sig0 + 8 * (j % NSIG), (uint32_t)((j / NSIG) & 1));
                const int64_t b = sigb[j % NSIG];
                if (b < 0) break;
                // the compute threads' Y stores (ordered before their arrive)
                // made visible at gpu scope, then counted
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctl.done_a + b) : "memory");
                *sigdone = j + 1;
            }
        }
        return;
    }

    // ---- compute warps (256 threads, named barrier 1) ----
    const int lo = tid & 15, hi = tid >> 4;
    int ja = 0;  // A tasks computed by this CTA
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
        const int64_t i = task[s];
        if (i >= ntasks) break;
        bool isb;
        int64_t b;
        int part;
        ab_decode<T>(i, batch, Dp, isb, b, part);
        if (!isb) {
            st_task_a<INV, N1>(st, lo, hi, 1, empty0 + 8 * s, part, ring + (b % ctl.ring) * L, scale, tw4, tw256,
                                  opts);
            if (tid == 0) sigb[ja % NSIG] = b;
            bk_arrive(sig0 + 8 * (ja % NSIG));  // release: this thread's Y stores
            ++ja;
        } else {
            // the stage's Y rows landed (the TMA read is complete): the ring
            // slot's rows are free for the next transform
            if (tid == 0) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctl.done_b + b) : "memory");
            if constexpr (L == 65536)
                st_task_b<INV>(st, lo, hi, 1, empty0 + 8 * s, out + b * 65536 + part * 16, tw256, opts);
            else
                st_task_b128<INV, OTW>(st, tid, 1, empty0 + 8 * s, out + b * L + part * ROWS, ow, b, part * ROWS);
        }
    }
    // done: tell the signaller (once its slot is free)
    if (tid == 0) {
        while (*sigdone < ja - NSIG + 1) __nanosleep(20);
        sigb[ja % NSIG] = -1;
    }
    grp_sync(1);
    bk_arrive(sig0 + 8 * (ja % NSIG));
}

}  // namespace b200fft
