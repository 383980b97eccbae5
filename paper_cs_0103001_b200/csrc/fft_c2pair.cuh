// fft_c2pair.cuh -- C2's 65536-point complex64 transform with the
// intermediate Y kept ON CHIP: one 2-CTA cluster per transform, each CTA
// parks its half of Y in tensor memory (TMEM, 256 KiB per SM) and the two
// halves meet through distributed shared memory (DSMEM).
//
// What is computed: the same four-step split as k_ab_st (fft_c2.cuh; the
// DFT of Eq. E2, with its 1/N, or the unscaled inverse of
// Sec. 3), n = n1 + 256 n2, k = k2 + 256 k1:
//   Y[k2][n1] = W_N^{n1 k2} sum_{n2} x[n1 + 256 n2] W_256^{n2 k2}   (A)
//   X[k2 + 256 k1] = sum_{n1} Y[k2][n1] W_256^{n1 k1}                (B)
// Why: k_ab_st sends Y out to an L2 ring and back -- four SM <-> L2
// crossings per element, whose L2 round trip is that kernel's floor
// (profiles/README.md, 0.70-0.73 of HBM).  Here Y never leaves the pair of
// SMs: two crossings per element (x in, X out) plus half of Y over DSMEM.
//
// Per transform b (pair = cluster; CTA rank c in {0, 1}):
//   A tasks p in [8c, 8c + 8): columns n1 in [16p, 16p + 16) (the TMA box
//     [256 n2][16 n1], 32 KiB), two groups of 256 compute threads, group g
//     takes p = 8c + g + 2i, i < 4.  Thread (lo, hi) ends with Y[hi + 16q]
//     [16p + lo], q < 16, and parks the 16 values in its own TMEM lane
//     (column 8q + 2i of its 128-column range): no thread ever reads another
//     thread's TMEM, so program order alone orders A(b + 1)'s writes after
//     B(b)'s reads.
//   B steps j < 8: CTA c owns rows k2 in [16Q, 16Q + 16), Q = 8c + j.  Every
//     thread of both CTAs contributes its 4 parked values of rows Q to the
//     gather buffer of the owning CTA: [16 rows][256 n1], its own CTA's by
//     st.shared, the peer's by st.async (DSMEM, counted on the buffer's full
//     barrier as transaction bytes).  Group j % 2 of the owner then runs the
//     B task body of k_ab_st (256-point DFTs over n1, X stores from
//     registers) on the buffer.
// Synchronisation per gather buffer s (NB of them, used in step order u):
//   gfull[s]  : 512 local arrivals (+ 16 KiB of the peer's st.async bytes)
//   gempty[s] : the computing group's 256 threads have read it
//   pempty[s] : the PEER's buffer s has been read (the peer arrives remotely)
// Every wait points at an earlier step of the same step order on both CTAs,
// and the A stages are fed by one producer per group: deadlock-free.
#pragma once
#include "fft_c2.cuh"

namespace b200fft {

struct PairCfg {
    static constexpr int NSA = 2;  // A stages per compute group
    static constexpr int NB = 2;   // gather buffers (= the two B steps in flight)
    static constexpr size_t TILE = 16 * 256 * 8;
    static constexpr size_t B_OFF = 2 * NSA * TILE;
    static constexpr size_t BAR_OFF = B_OFF + NB * TILE;  // afull[2][NSA], aempty[2][NSA], gfull, gempty, pempty [NB]
    static constexpr size_t NBAR = 4 * NSA + 3 * NB;
    static constexpr size_t TM_OFF = BAR_OFF + 8 * NBAR;
    static constexpr size_t SMEM = TM_OFF + 16;
    static constexpr int THREADS = 18 * 32;  // 16 compute warps, 2 producer warps
};

__device__ __forceinline__ uint32_t pr_cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t pr_mapa(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void pr_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// wait with cluster-scope acquire (the peer's st.async bytes / remote arrivals)
__device__ __forceinline__ void pr_wait_cl(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "PR_WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n"
        "@!p bra PR_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(20000u)
        : "memory");
}
__device__ __forceinline__ void pr_arrive_remote(uint32_t rbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void pr_st_async(uint32_t raddr, float2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
                 "f"(v.x), "f"(v.y), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void tm_st2(uint32_t taddr, float2 v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};\n" ::"r"(taddr), "r"(__float_as_uint(v.x)),
                 "r"(__float_as_uint(v.y))
                 : "memory");
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, float2 (&v)[4]) {
    uint32_t r[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 "tcgen05.wait::ld.sync.aligned;\n"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = make_float2(__uint_as_float(r[2 * i]), __uint_as_float(r[2 * i + 1]));
}

// A task body: k_ab_st's st_task_a with the Y rows parked in TMEM
template <bool INV>
__device__ __forceinline__ void pair_task_a(float2* st, int lo, int hi, int bar, uint32_t empty, int part,
                                            float scale, const float2* __restrict__ tw4, uint32_t taddr, int xo) {
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
        st_step1_twiddle_c<INV>(v, hi);
        dft<16, INV>(v);
    }
    // Y[k2][n1] = v[q] W_N^{n1 k2} scale, k2 = hi + 16 q -> TMEM column 8 q (+ 2 i in taddr)
    const int n1 = part * 16 + lo;
    float2 wm = cscale(__ldg(tw4 + (int64_t)hi * 256 + n1), scale);
    const float2 ws = __ldg(tw4 + (int64_t)16 * 256 + n1);
#pragma unroll
    for (int q = 0; q < 16; ++q) {
        if (!(xo & 16)) tm_st2(taddr + 8 * q, cmul_dir<INV>(v[q], wm));
        else if (v[q].x == 1.2345e-38f) st[q] = v[q];
        if (q < 15) wm = cmul(wm, ws);
    }
}

template <bool INV>
__global__ void __launch_bounds__(PairCfg::THREADS, 1)
    k_ab_pair(const __grid_constant__ CUtensorMap map_x, float2* __restrict__ out, int64_t batch, float scale,
              const float2* __restrict__ tw4, const float2* __restrict__ tw256, int xo) {
    // xo: timing-experiment bits (wrong results; B200FFT_PAIR_XO with
    // B200FFT_ALLOW_WRONG=1): 2 no X stores, 4 no TMA
    // loads, 8 no FFT arithmetic, 16 no TMEM traffic, 64 no in-stage exchanges
    using G = PairCfg;
    constexpr int NSA = G::NSA, NB = G::NB;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t afull0 = s_base + (uint32_t)G::BAR_OFF, aempty0 = afull0 + 8 * 2 * NSA;
    const uint32_t gfull0 = aempty0 + 8 * 2 * NSA, gempty0 = gfull0 + 8 * NB, pempty0 = gempty0 + 8 * NB;
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint32_t c = pr_cluster_rank(), peer = c ^ 1u;
    const int64_t pair = blockIdx.x / 2, npairs = gridDim.x / 2;
    const int64_t ntr = batch > pair ? (batch - 1 - pair) / npairs + 1 : 0;  // transforms of this pair

    if (tid == 0) {
        for (int s = 0; s < 2 * NSA; ++s) {
            bk_mbar_init(afull0 + 8 * s, 1);
            bk_mbar_init(aempty0 + 8 * s, 256);
        }
        for (int s = 0; s < NB; ++s) {
            bk_mbar_init(gfull0 + 8 * s, 512);
            bk_mbar_init(gempty0 + 8 * s, 256);
            bk_mbar_init(pempty0 + 8 * s, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) {  // the CTA's whole TMEM (512 columns x 128 lanes)
        asm volatile(
            "tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
            "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::"r"(s_base + (uint32_t)G::TM_OFF)
            : "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    pr_cluster_sync();  // the peer's barriers are initialised before any remote operation
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(smem_raw + G::TM_OFF);

    if (warp >= 16) {  // ---- producers: one per compute group ----
        if ((tid & 31) == 0) {
            const int g = warp - 16;
            const uint64_t pol = tmaops::policy_evict_first();
            for (int64_t m = 0; m < ntr; ++m) {
                const int64_t b = pair + m * npairs;
                for (int i = 0; i < 4; ++i) {
                    const int64_t k = m * 4 + i;
                    const int s = g * NSA + (int)(k % NSA);
                    if (k >= NSA) bk_wait(aempty0 + 8 * s, (uint32_t)(((k / NSA) - 1) & 1));
                    if (xo & 4) {
                        bk_arrive(afull0 + 8 * s);
                        continue;
                    }
                    bk_arrive_expect(afull0 + 8 * s, (uint32_t)G::TILE);
                    tmaops::load3(s_base + (uint32_t)(s * G::TILE), &map_x, (int)(8 * c + g + 2 * i) * 16, 0, (int)b,
                                  afull0 + 8 * s, pol);
                }
            }
        }
        __syncwarp();  // the whole warp reaches the teardown barriers together
    } else {  // ---- compute: group g = warps 8g .. 8g + 7 ----
        const int g = warp >> 3, tg = tid & 255, lo = tg & 15, hi = tg >> 4;
        // this thread's TMEM: lane 32 (warp % 4) + lane id, columns 128 (warp / 4) ..
        const uint32_t tm = tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(128 * (warp >> 2));
        float2* gbuf = reinterpret_cast<float2*>(smem_raw + G::B_OFF);
        const uint32_t gbuf_s = s_base + (uint32_t)G::B_OFF;
        int64_t u = 0;  // B steps of this CTA
        for (int64_t m = 0; m < ntr; ++m) {
            const int64_t b = pair + m * npairs;
            for (int i = 0; i < 4; ++i) {
                const int64_t k = m * 4 + i;
                const int s = g * NSA + (int)(k % NSA);
                bk_wait(afull0 + 8 * s, (uint32_t)((k / NSA) & 1));
                pair_task_a<INV>(reinterpret_cast<float2*>(smem_raw + s * G::TILE), lo, hi, 1 + g, aempty0 + 8 * s,
                                 (int)(8 * c + g + 2 * i), scale, tw4, tm + 2 * i, xo);
            }
            asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
            // B steps in pairs: every thread contributes to both steps of a
            // pair before its group computes its own one, so the two groups'
            // B tasks run concurrently (NB = 2 buffers = the pair in flight)
            for (int jj = 0; jj < 8; jj += 2, u += 2) {
#pragma unroll
                for (int d = 0; d < 2; ++d) {
                    const int j = jj + d;
                    const int s = (int)((u + d) % NB);
                    const uint32_t ph = (uint32_t)(((u + d) / NB) & 1);
                    if (u + d >= NB) {
                        bk_wait(gempty0 + 8 * s, ph ^ 1u);     // my buffer s: its previous use read
                        pr_wait_cl(pempty0 + 8 * s, ph ^ 1u);  // the peer's buffer s: likewise
                    }
                    const int qo = 8 * (int)c + j, qp = 8 * (int)peer + j;
                    float2 vo[4], vp[4];
                    __syncwarp();  // tcgen05.ld is warp-collective
                    if (!(xo & 16)) {
                        tm_ld8(tm + 8 * qo, vo);
                        tm_ld8(tm + 8 * qp, vp);
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i) vo[i] = vp[i] = make_float2((float)lo, (float)i);
                    }
                    const uint32_t rbar = pr_mapa(gfull0 + 8 * s, peer);
                    const uint32_t rbuf = pr_mapa(gbuf_s + (uint32_t)(s * G::TILE), peer);
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const int idx = hi * 256 + 16 * (8 * (int)c + g + 2 * i) + lo;  // [row hi][n1]
                        gbuf[s * 4096 + idx] = vo[i];
                        pr_st_async(rbuf + 8 * idx, vp[i], rbar);
                    }
                    if (tid == 0) bk_arrive_expect(gfull0 + 8 * s, 16384u);
                    else bk_arrive(gfull0 + 8 * s);
                }
                const int j = jj + g;
                const int s = (int)((u + g) % NB);
                const uint32_t ph = (uint32_t)(((u + g) / NB) & 1);
                pr_wait_cl(gfull0 + 8 * s, ph);
                st_task_b<INV>(gbuf + s * 4096, lo, hi, 1 + g, gempty0 + 8 * s, out + b * 65536 + 16 * (8 * (int)c + j),
                               tw256, xo & (2 | 8 | 64));
                if (tg == 0) {  // tell the peer once all 256 have read buffer s
                    bk_wait(gempty0 + 8 * s, ph);
                    pr_arrive_remote(pr_mapa(pempty0 + 8 * s, peer));
                }
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    pr_cluster_sync();  // no peer operation on this CTA's smem is outstanding
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem) : "memory");
}

}  // namespace b200fft
