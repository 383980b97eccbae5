// fft_colpipe.cuh -- the column direction of the separable Gaussian
// pipeline for 8192-long columns (C4 = BASELINE configs[3]) in ONE HBM pass.
//
// What is computed (eq5 / 2D-IDFT, P:377-381 the filter): for
// every column v of an N x M grid (N = 8192 = 64 x 128), the column operator
//     f -> IDFT_N( g_N(u) / N . DFT_N(f) )          (Gaussian, u signed index)
// by the four-step split x = n2 + 128 n1, u = k1 + 64 k2 (n1, k1 < 64;
// n2, k2 < 128), in place on the grid:
//   A  (n2, v): Y[k1][n2] = W_N^{n2 k1} sum_{n1} f[n2 + 128 n1] W_64^{n1 k1}
//               (stored at row n2 + 128 k1)
//   B  (k1, v): 128-point forward over n2 -> k2, x g_N[k1 + 64 k2] / N
//               (x g_M[v + col_off] for a distributed column slab), 128-point
//               inverse back over k2 -> n2 (rows 128 k1 .. 128 k1 + 127)
//   A' (n2, v): conj twiddle W_N^{-n2 k1}, 64-point inverse over k1 -> n1
// -- the same sums as the three k_cols passes (MODE 3, MODE 2 kind 6 / 7,
// MODE 4), each of which streams the whole grid through HBM.  Here a group
// g = 16 adjacent columns x all N rows (1 MiB) goes through A, B and A' as
// 3 x 32 tasks of 32 KiB while it stays in L2 (outputs stored with an
// evict_last hint), so HBM sees one read and one write of the grid.
//
// Scheduling = k_ab_st's (fft_c2.cuh): positions of a global order handed
// out by an atomic counter; block j holds A(j) | B(j - D) | A'(j - 2D) (32
// tasks each); B(g) waits for A(g)'s 32 signals, A'(g) for B(g)'s; a
// signaller warp makes each A / B task's stores visible at gpu scope
// (fence.acq_rel.gpu) before counting it.  All waits point back in the
// order and no signal waits for a later load: deadlock-free with all CTAs
// co-resident (cooperative launch).
#pragma once
#include "fft_c2.cuh"

namespace b200fft {

struct ColPipeCtl {
    int* done_a;               // [groups] A tasks whose outputs are visible
    int* done_b;               // [groups] B tasks whose outputs are visible
    unsigned long long* next;  // next position
    int D;                     // phase distance (blocks)
};

struct ColPipeCfg {
    static constexpr int NS = 2, NSIG = 4;
    static constexpr size_t STAGE = 32768;
    static constexpr size_t BAR_OFF = NS * STAGE;                        // full[NS], empty[NS], sig[NSIG]
    static constexpr size_t INFO_OFF = BAR_OFF + 8 * (2 * NS + NSIG);    // task[NS], sigb[NSIG] (int64), sigdone
    static constexpr size_t SMEM = INFO_OFF + 8 * (NS + NSIG) + 16;
};

// position -> (phase 0 = A, 1 = B, 2 = A', group, part); false for the
// empty slots of the ramp-up / ramp-down blocks
__device__ __forceinline__ bool cp_decode(int64_t p, int64_t G, int D, int& phase, int64_t& g, int& part) {
    // positions < 2^31 (launch_colfilt bounds the group count): 32-bit division
    const int64_t j = (int64_t)((uint32_t)p / 96u);
    const int r = (int)((uint32_t)p - (uint32_t)j * 96u);
    phase = r / 32;
    part = r % 32;
    g = j - (int64_t)phase * D;
    return g >= 0 && g < G;
}

// group g -> (image, first column): shift / mask for a power-of-two number
// of column groups per image (P2), else a 32-bit division (a separate
// instantiation: the division's registers pushed the B task into spills)
template <bool P2>
__device__ __forceinline__ void cp_group(int64_t g, int64_t CG, int cg_sh, int& img, int& c0) {
    if constexpr (P2) {
        img = (int)(g >> cg_sh);
        c0 = (int)(g & (CG - 1)) * 16;
    } else {
        img = (int)((uint32_t)g / (uint32_t)CG);
        c0 = (int)((uint32_t)g - (uint32_t)img * (uint32_t)CG) * 16;
    }
}

// grid: [nimg][8192][M] complex64 (in place); tl = W_N^x, x < N (fp64-generated);
// gu = g_N[u] (N entries); gv = g_M (M_total entries, distributed slabs) or null
template <int N2 = 128, int TW = 0, bool P2 = true>
__global__ void __launch_bounds__(320, 3)
    k_colfilt(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
              float2* __restrict__ grid, int64_t M, int64_t nimg, float scale, const float2* __restrict__ tw64,
              const float2* __restrict__ tw128, const float2* __restrict__ tl, const float* __restrict__ gu,
              const float* __restrict__ gv, int64_t col_off, int cg_sh, ColPipeCtl ctl) {
    using G = ColPipeCfg;
    constexpr int NS = G::NS, NSIG = G::NSIG;
    constexpr int64_t N = 64 * N2;
    static_assert(N2 == 128, "A / A' tasks cover 4 of the 128 n2 values");
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, empty0 = full0 + 8 * NS, sig0 = empty0 + 8 * NS;
    volatile int64_t* task = reinterpret_cast<volatile int64_t*>(smem_raw + G::INFO_OFF);
    volatile int64_t* sigb = task + NS;
    volatile int* sigdone = reinterpret_cast<volatile int*>(sigb + NSIG);
    const int tid = threadIdx.x;
    const int64_t CG = M / 16;  // column groups per image (2^cg_sh, or cg_sh = -1)
    const int64_t groups = CG * nimg;
    const int64_t npos = (groups + 2 * (int64_t)ctl.D) * 96;

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
        if ((tid & 31) != 0) return;
        if (tid < 288) {  // ---- producer ----
            const uint64_t pol_stream = tmaops::policy_evict_first();
            const uint64_t pol_keep = tmaops::policy_evict_last();
            int na = 0;  // signal-producing (A, B) tasks issued
            for (int64_t k = 0;; ++k) {
                const int s = (int)(k % NS);
                if (k >= NS) bk_wait(empty0 + 8 * s, (uint32_t)(((k / NS) - 1) & 1));
                int phase = 0, part = 0;
                int64_t g = 0, i;
                do {  // skip the ramp's empty slots
                    i = (int64_t)atomicAdd(ctl.next, 1ull);
                } while (i < npos && !cp_decode(i, groups, ctl.D, phase, g, part));
                const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
                if (i >= npos) {
                    task[s] = -1;
                    bk_arrive(bar);
                    break;
                }
                task[s] = i;
                int img, c0;
                cp_group<P2>(g, CG, cg_sh, img, c0);
                if (phase != 2) {
                    while (*sigdone < na - NSIG + 1) __nanosleep(20);
                    ++na;
                }
                if (phase == 1) {
                    while (bk_ld_acquire(ctl.done_a + g) < 32) __nanosleep(32);
                } else if (phase == 2) {
                    while (bk_ld_acquire(ctl.done_b + g) < 32) __nanosleep(32);
                }
                if (phase != 0) asm volatile("fence.proxy.async.global;\n" ::: "memory");
                bk_arrive_expect(bar, (uint32_t)G::STAGE);
                if (phase == 1)  // rows 128 k1 .. for k1 = 2 part, 2 part + 1: [256][16]
                    tmaops::load3(st, &map_b, c0, (int)(img * N + 256 * part), 0, bar, pol_keep);
                else  // rows n2 + 128 n1, n2 = 4 part .. 4 part + 3: [64 n1][4][16]
                    tmaops::load3(st, &map_a, c0, 4 * part, img * 64, bar, phase == 0 ? pol_stream : pol_keep);
            }
        } else {  // ---- signaller ----
            for (int j = 0;; ++j) {
                bk_wait(sig0 + 8 * (j % NSIG), (uint32_t)((j / NSIG) & 1));
                const int64_t code = sigb[j % NSIG];
                if (code < 0) break;
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                int* ctr = ((code & 1) ? ctl.done_b : ctl.done_a) + (code >> 1);
                asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctr) : "memory");
                *sigdone = j + 1;
            }
        }
        return;
    }

    // ---- compute warps (256 threads, named barrier 1) ----
    // step twiddles from the constant table (TWREC 2): lt = tid / 64 (A, A')
    // or tid / 32 (B) is uniform across a warp
    // (TW bit 0: A / A' steps, bit 1: B steps from the constant table)
    using FA = LineFFT<float, 64, 16, false, 5, false, (TW & 1) ? 2 : 1>;
    using FAI = LineFFT<float, 64, 16, true, 5, false, (TW & 1) ? 2 : 1>;
    using FB = LineFFT<float, 128, 16, false, 2, false, (TW & 2) ? 2 : 1>;
    using FBI = LineFFT<float, 128, 16, true, 2, false, (TW & 2) ? 2 : 1>;
    const uint64_t keep = tmaops::policy_evict_last();
    const uint64_t stream = tmaops::policy_evict_first();
    int ja = 0;
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
        const int64_t i = task[s];
        if (i < 0) break;
        int phase, part;
        int64_t g;
        cp_decode(i, groups, ctl.D, phase, g, part);
        int img_i, c0_i;
        cp_group<P2>(g, CG, cg_sh, img_i, c0_i);
        const int64_t img = img_i, c0 = c0_i;
        float2 v[16];
        if (phase != 1) {
            // line (n2l, col) = tid % 64, 4 lanes of 16 elements (n1 or k1)
            const int line = tid & 63, lt = tid >> 6;
            const int n2l = line >> 4, col = line & 15;
            const int64_t n2 = 4 * part + n2l;
            float2* ln = st + line;
            // W_N^{n2 (lt + 4 m)} = W_N^{n2 lt} (W_N^{4 n2})^m
            float2 wm = __ldg(tl + n2 * lt);
            const float2 ws = __ldg(tl + n2 * 4);
            float2* o = grid + (img * N + n2) * M + c0 + col;
            if (phase == 0) {
#pragma unroll
                for (int m = 0; m < 16; ++m) v[FA::pos_in(m)] = ln[FA::bpos(lt, m)];
                FA::run(v, ln, lt, tw64, -256);
                bk_arrive(empty0 + 8 * s);
#pragma unroll
                for (int m = 0; m < 16; ++m) {  // element k1 = lt + 4 m -> row n2 + 128 k1
                    st_pol(o + (int64_t)(lt + 4 * m) * 128 * M, cmul(v[FA::pos_out(m)], wm), keep);
                    wm = cmul(wm, ws);
                }
            } else {
#pragma unroll
                for (int m = 0; m < 16; ++m) {  // element k1 = lt + 4 m, times conj W_N^{n2 k1}
                    v[FAI::pos_in(m)] = cmulc(ln[FAI::bpos(lt, m)], wm);
                    wm = cmul(wm, ws);
                }
                FAI::run(v, ln, lt, tw64, -256);
                bk_arrive(empty0 + 8 * s);
#pragma unroll
                for (int m = 0; m < 16; ++m)  // element n1 = lt + 4 m -> row n2 + 128 n1
                    st_pol(o + (int64_t)(lt + 4 * m) * 128 * M, v[FAI::pos_out(m)], stream);
            }
        } else {
            // line (k1l, col) = tid % 32, 8 lanes of 16 elements (n2, then k2)
            const int line = tid & 31, lt = tid >> 5;
            const int k1l = line >> 4, col = line & 15;
            const int64_t k1 = 2 * part + k1l;
            float2* ln = st + k1l * 2048 + col;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FB::pos_in(m)] = ln[FB::bpos(lt, m)];
            FB::run(v, ln, lt, tw128, -256);
            float hcol = scale;
            if (gv) hcol *= __ldg(gv + col_off + c0 + col);
            float2 w[16];
#pragma unroll
            for (int m = 0; m < 16; ++m)  // element k2 = lt + 8 m: u = k1 + 64 k2
                w[FBI::pos_in(m)] = cscale(v[FB::pos_out(m)], __ldg(gu + k1 + 64 * (lt + 8 * m)) * hcol);
            FBI::run(w, ln, lt, tw128, -256);
            bk_arrive(empty0 + 8 * s);
            float2* o = grid + (img * N + 128 * k1) * M + c0 + col;
#pragma unroll
            for (int m = 0; m < 16; ++m)  // element n2 = lt + 8 m -> row 128 k1 + n2
                st_pol(o + (int64_t)(lt + 8 * m) * M, w[FBI::pos_out(m)], keep);
        }
        if (phase != 2) {
            if (tid == 0) sigb[ja % NSIG] = 2 * g + (phase == 1 ? 1 : 0);
            bk_arrive(sig0 + 8 * (ja % NSIG));  // release: this thread's stores
            ++ja;
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
