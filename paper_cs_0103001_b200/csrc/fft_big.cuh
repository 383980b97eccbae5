// fft_big.cuh -- one complex64 transform of n = 2^30 (C5 = BASELINE
// configs[4] on one GPU) in TWO HBM passes instead of four.
//
// What is computed: the DFT of Eq. E2 with its 1/n, or the
// unscaled inverse of Eq. E3 / Sec. 3, by the four-step
// split n = N1 N2 (N1 = N2 = 32768), x[n1 + N1 n2], X[k2 + N2 k1] -- the
// first factorisation of the paper's cyclic split with N1 = N2:
//   pass 1: for every column n1, the 32768-point DFT over n2 -> k2, times
//           W_n^{n1 k2} (the four-step twiddle): Y[k2][n1]
//   pass 2: for every row k2 of Y, the 32768-point DFT over n1 -> k1, times
//           the paper's 1/n (forward): X[k2 + N2 k1]
// Each 32768-point line transform is itself the inner four-step
// l = a + 128 c, k = kc + 256 ka (a, ka < 128; c, kc < 256):
//   A (per a):  256-point DFT over c -> kc, times W_L^{a kc}   (L = 32768)
//   B (per kc): 128-point DFT over a -> ka
// with the A -> B intermediate in an L2-resident ring (as in fft_c2.cuh):
// a GROUP is 16 adjacent lines (pass 1: columns n1, so every HBM access is a
// 128-B run; pass 2: rows k2, so the strided X stores are 128-B runs too) --
// 16 x 32768 x 8 B = 4 MiB per ring slot; 128 A tasks and 128 B tasks of
// 32 KiB per group.
//   pass 1 A (group g, a):  TMA box [256 c][16 n1] (rows a + 128 c); line = n1
//           -> ring[slot][kc][a][16 n1]
//   pass 1 B (group g, kc pair): box [2 kc][128 a][16 n1]; lines (kc, n1);
//           x W_n^{n1 k2}, k2 = kc + 256 ka -> Y[k2][n1] (16 n1 = 128 B)
//   pass 2 A (group g, row r, a block of 16): box [256 c][16 a] of row k2 =
//           16 g + r; line = a -> ring[slot][kc][r][a] (16 a = 128 B)
//   pass 2 B (group g, kc pair): box [2 kc][16 r][128 a] (lines contiguous):
//           step 0 with 8 lanes per line, exchange through the XOR layout
//           x * 32 + (line ^ 4 (x / 16 mod 4)), step 1 line-fastest;
//           x 1/n -> X[(16 g + r) + N2 (kc + 256 ka)] (16 rows = 128 B)
// Scheduling, signals and deadlock freedom: those of k_ab_st (dynamic
// positions A(j) | B(j - D), 256 per block; a signaller per CTA; an A task
// reuses a ring slot only after the B tasks of its previous group).
#pragma once
#include "fft_c2.cuh"

namespace b200fft {

struct BigCtl {
    int* done_a;               // [groups] A tasks whose ring rows are visible
    int* done_b;               // [groups] B tasks that have read their ring rows
    unsigned long long* next;  // next position
    int D, ring;               // phase distance (groups), ring slots
};

struct BigCfg {
    static constexpr int NS = 2, NSIG = 4;
    static constexpr size_t STAGE = 32768;
    static constexpr size_t BAR_OFF = NS * STAGE;                       // full[NS], empty[NS], sig[NSIG]
    static constexpr size_t INFO_OFF = BAR_OFF + 8 * (2 * NS + NSIG);   // task[NS], sigb[NSIG] (int64), sigdone
    static constexpr size_t SMEM = INFO_OFF + 8 * (NS + NSIG) + 16;
    static constexpr int64_t L = 32768;                                 // line length (both passes)
    static constexpr int64_t SLOT = 16 * L;                             // ring slot (elements)
};

// position -> (B?, group, part), 256 positions per block: A(j) 128 | B(j - D) 128
__device__ __forceinline__ bool big_decode(int64_t p, int64_t G, int D, bool& isb, int64_t& g, int& part) {
    const int64_t j = p >> 8;
    const int r = (int)(p & 255);
    isb = r >= 128;
    part = r & 127;
    g = j - (isb ? D : 0);
    return g >= 0 && g < G;
}

// W_n^x for x < 2^30 from two fp64-generated tables: hi[x >> 15] lo[x & 32767]
// (pass 1's B tasks; the product is formed after the FFT, the loads before)

// pass 2's B exchange uses big_bx (fft_c2.cuh): element x of line L at
// x * 32 + (L ^ 2 ((x / 16) mod 8)) -- the line XOR 4 ((x / 16) mod 4) had
// 2-way conflicts on every write (ncu: 209 M excess wavefronts per pass).

template <bool INV, int PASS>
__global__ void __launch_bounds__(320, 3)
    k_big(const __grid_constant__ CUtensorMap map_in, const __grid_constant__ CUtensorMap map_ring,
          float2* __restrict__ ring, float2* __restrict__ out, float scale, const float2* __restrict__ tw256,
          const float2* __restrict__ tw128, const float2* __restrict__ twl, const float2* __restrict__ whi,
          const float2* __restrict__ wlo, BigCtl ctl, int xo) {
    using G = BigCfg;
    constexpr int NS = G::NS, NSIG = G::NSIG;
    constexpr int64_t L = G::L, GROUPS = 2048;  // 32768 lines / 16
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    const uint32_t s_base = (uint32_t)__cvta_generic_to_shared(smem_raw);
    const uint32_t full0 = s_base + (uint32_t)G::BAR_OFF, empty0 = full0 + 8 * NS, sig0 = empty0 + 8 * NS;
    volatile int64_t* task = reinterpret_cast<volatile int64_t*>(smem_raw + G::INFO_OFF);
    volatile int64_t* sigb = task + NS;
    volatile int* sigdone = reinterpret_cast<volatile int*>(sigb + NSIG);
    const int tid = threadIdx.x;
    const int64_t npos = (GROUPS + ctl.D) * 256;

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
            int na = 0;
            for (int64_t k = 0;; ++k) {
                const int s = (int)(k % NS);
                if (k >= NS) bk_wait(empty0 + 8 * s, (uint32_t)(((k / NS) - 1) & 1));
                bool isb = false;
                int part = 0;
                int64_t g = 0, i;
                do {
                    i = (int64_t)atomicAdd(ctl.next, 1ull);
                } while (i < npos && !big_decode(i, GROUPS, ctl.D, isb, g, part));
                const uint32_t st = s_base + (uint32_t)(s * G::STAGE), bar = full0 + 8 * s;
                if (i >= npos) {
                    task[s] = -1;
                    bk_arrive(bar);
                    break;
                }
                task[s] = i;
                const int slot = (int)(g % ctl.ring);
                if (!isb) {
                    while (*sigdone < na - NSIG + 1) __nanosleep(20);
                    ++na;
                    if (g >= ctl.ring)  // the slot's previous group: all its B tasks have read it
                        while (bk_ld_acquire(ctl.done_b + (g - ctl.ring)) < 128) __nanosleep(32);
                    bk_arrive_expect(bar, (uint32_t)G::STAGE);
                    if (PASS == 1)  // rows a + 128 c, columns 16 g .. : [256 c][16]
                        tmaops::load3(st, &map_in, (int)(16 * g), part, 0, bar, pol_stream);
                    else  // row 16 g + r, elements a + 128 c, a in [16 ab, +16): [256 c][16 a]
                        tmaops::load3(st, &map_in, 16 * (part & 7), 0, (int)(16 * g + (part >> 3)), bar, pol_stream);
                } else {
                    while (bk_ld_acquire(ctl.done_a + g) < 128) __nanosleep(32);
                    asm volatile("fence.proxy.async.global;\n" ::: "memory");
                    bk_arrive_expect(bar, (uint32_t)G::STAGE);
                    // kc = 2 part, 2 part + 1 of the slot: 32 KiB contiguous
                    // (view {16 | 128, 128 | 16, 256 ring}: box [2 kc][..][..])
                    tmaops::load3(st, &map_ring, 0, 0, slot * 256 + 2 * part, bar, pol_keep);
                }
            }
        } else {  // ---- signaller ----
            for (int j = 0;; ++j) {
                bk_wait(sig0 + 8 * (j % NSIG), (uint32_t)((j / NSIG) & 1));
                const int64_t g = sigb[j % NSIG];
                if (g < 0) break;
                asm volatile("fence.acq_rel.gpu;\n" ::: "memory");
                asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctl.done_a + g) : "memory");
                *sigdone = j + 1;
            }
        }
        return;
    }

    // ---- compute warps (256 threads, named barrier 1) ----
    // step twiddles from the constant table (TWREC 2): the butterfly index is
    // the lane index hi (A: two values per warp) or lt = tid / 32 (B: one)
    using FA = LineFFT<float, 256, 16, INV, 2, false, 2>;
    using FB = LineFFT<float, 128, 16, INV, 2, false, 2>;
    const uint64_t keep = tmaops::policy_evict_last();
    const uint64_t stream = tmaops::policy_evict_first();
    const int lo = tid & 15, hi = tid >> 4;
    int ja = 0;
    for (int64_t k = 0;; ++k) {
        const int s = (int)(k % NS);
        float2* st = reinterpret_cast<float2*>(smem_raw + s * G::STAGE);
        bk_wait(full0 + 8 * s, (uint32_t)((k / NS) & 1));
        const int64_t i = task[s];
        if (i < 0) break;
        bool isb;
        int part;
        int64_t g;
        big_decode(i, GROUPS, ctl.D, isb, g, part);
        float2* slot = ring + (g % ctl.ring) * G::SLOT;
        float2 v[16];
        if (!isb) {
            // line t = lo (pass 1: column n1 = 16 g + t; pass 2: a = 16 ab + t),
            // elements c = hi + 16 r of the [256 c][16] box
            const int a = PASS == 1 ? part : 16 * (part & 7) + lo;
            // W_L^{a kc}, kc = hi + 16 m: W_L^{a hi} (W_L^{16 a})^m; pass 2 forward also the 1/n
            // (loaded before the FFT: their latency hides behind it)
            float2 wm = __ldg(twl + a * hi);
            const float2 ws = __ldg(twl + 16 * a);
            float2* ln = st + lo;
#pragma unroll
            for (int m = 0; m < 16; ++m) v[FA::pos_in(m)] = ln[FA::bpos(hi, m)];
            FA::run(v, ln, hi, tw256, -256);
            bk_arrive(empty0 + 8 * s);
            if (PASS == 2) wm = cscale(wm, scale);
            // pass 1: ring[kc][a][16 n1]; pass 2: ring[kc][r][128 a]
            // (pass 2: line (kc, r) stored with element a at a ^ 8 (r mod 4), so
            // the B task's step-0 reads of 4 lines per warp hit distinct banks)
            float2* y = PASS == 1 ? slot + (int64_t)hi * 2048 + a * 16 + lo
                                  : slot + (int64_t)hi * 2048 + (part >> 3) * 128 + (a ^ (8 * ((part >> 3) & 3)));
#pragma unroll
            for (int m = 0; m < 16; ++m) {
                st_pol(y + m * 16 * 2048, cmul_dir<INV>(v[FA::pos_out(m)], wm), keep);
                wm = cmul(wm, ws);
            }
            if (tid == 0) sigb[ja % NSIG] = g;
            bk_arrive(sig0 + 8 * (ja % NSIG));
            ++ja;
        } else {
            // the stage's ring rows landed: the slot's rows are read
            if (tid == 0) asm volatile("red.relaxed.gpu.global.add.s32 [%0], 1;\n" ::"l"(ctl.done_b + g) : "memory");
            const int line = tid & 31, lt = tid >> 5;  // line (kcl, t), 8 lanes of 16 elements
            const int kcl = line >> 4, t = line & 15;
            const int64_t kc = 2 * part + kcl;
            if (PASS == 1) {
                // Y[k2][n1] x W_n^{n1 k2}, k2 = kc + 256 ka, ka = lt + 8 m:
                // W_n^{n1 (kc + 256 lt)} (W_n^{2048 n1})^m -- the four table
                // entries loaded before the FFT (latency hidden behind it)
                const int64_t n1 = 16 * g + t;
                const int64_t x0 = n1 * (kc + 256 * lt), x1 = n1 * 2048;
                const float2 h0 = __ldg(whi + (x0 >> 15)), l0 = __ldg(wlo + (x0 & 32767));
                const float2 h1 = __ldg(whi + (x1 >> 15)), l1 = __ldg(wlo + (x1 & 32767));
                // [2 kc][128 a][16 n1]: element a of line (kcl, n1) at kcl 2048 + a 16 + n1
                float2* ln = st + kcl * 2048 + t;
#pragma unroll
                for (int m = 0; m < 16; ++m) v[FB::pos_in(m)] = ln[FB::bpos(lt, m)];
                FB::run(v, ln, lt, tw128, -256);
                bk_arrive(empty0 + 8 * s);
                float2 wm = cmul(h0, l0);
                const float2 ws = cmul(h1, l1);
                float2* o = out + (kc + 256 * lt) * L + n1;
                if (xo & 16) {  // timing experiment (wrong order): one contiguous 32 KiB block per task
                    float2* oc = out + (g * 128 + part) * 4096 + (lt * 16) * 32 + line;
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        oc[m * 32] = cmul_dir<INV>(v[FB::pos_out(m)], wm);
                        wm = cmul(wm, ws);
                    }
                } else if (xo & 2) {
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        o[(int64_t)m * 2048 * L] = cmul_dir<INV>(v[FB::pos_out(m)], wm);
                        wm = cmul(wm, ws);
                    }
                } else {
                    const uint64_t yp = (xo & 1) ? stream : keep;
#pragma unroll
                    for (int m = 0; m < 16; ++m) {
                        st_pol(o + (int64_t)m * 2048 * L, cmul_dir<INV>(v[FB::pos_out(m)], wm), yp);
                        wm = cmul(wm, ws);
                    }
                }
            } else {
                // [2 kc][16 r][128 a]: lines contiguous.  Step 0 (radix 16,
                // span 1): line L = tid / 8, lane j = tid % 8, elements j + 8 r
                const int L0 = tid >> 3, j = tid & 7;
                const float2* src = st + L0 * 128 + j;
                const int sw = L0 & 3;  // line stored with element a at a ^ 8 sw
#pragma unroll
                for (int r = 0; r < 16; ++r) v[r] = src[8 * (r ^ sw)];
                dft<16, INV>(v);
                grp_sync(1);
                // b[16 j + q] of line L0 -> XOR layout
#pragma unroll
                for (int q = 0; q < 16; ++q) st[big_bx(16 * j + q, L0)] = v[q];
                grp_sync(1);
                // step 1 (radix 8, span 16), line-fastest: line = tid % 32,
                // butterflies j' = lt + 8 b (b < 2): inputs b[j' + 16 r] W_128^{j' r}
                float2* u = v;  // step 0's values are in the stage now
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const int jp = lt + 8 * b;
#pragma unroll
                    for (int r = 0; r < 8; ++r) u[b * 8 + r] = st[big_bx(jp + 16 * r, line)];
                }
                bk_arrive(empty0 + 8 * s);
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const int jp = lt + 8 * b;
                    // W_128^{jp r} = W_256^{2 jp r} from the constant table (jp is warp-uniform)
#pragma unroll
                    for (int r = 1; r < 8; ++r) u[b * 8 + r] = cmul_dir<INV>(u[b * 8 + r], c_w256[(2 * jp * r) & 255]);
                    dft<8, INV>(u + b * 8);
                }
                // outputs c[jp + 16 q] = u[b 8 + q]: ka = jp + 16 q -> X[k2 + N2 (kc + 256 ka)]
                const int64_t k2 = 16 * g + t;
                float2* o = out + k2 + L * kc;
                if (xo & 4) {  // timing experiment (wrong order): one contiguous 32 KiB block per task
                    float2* oc = out + (g * 128 + part) * 4096 + line;
#pragma unroll
                    for (int b = 0; b < 2; ++b)
#pragma unroll
                        for (int q = 0; q < 8; ++q) oc[(lt + 8 * b + 16 * q) * 32] = u[b * 8 + q];
                } else if (xo & 8) {  // X without a cache hint
#pragma unroll
                    for (int b = 0; b < 2; ++b)
#pragma unroll
                        for (int q = 0; q < 8; ++q) o[(int64_t)(lt + 8 * b + 16 * q) * 256 * L] = u[b * 8 + q];
                } else {
#pragma unroll
                    for (int b = 0; b < 2; ++b)
#pragma unroll
                        for (int q = 0; q < 8; ++q)
                            st_pol(o + (int64_t)(lt + 8 * b + 16 * q) * 256 * L, u[b * 8 + q], stream);
                }
            }
        }
    }
    if (tid == 0) {
        while (*sigdone < ja - NSIG + 1) __nanosleep(20);
        sigb[ja % NSIG] = -1;
    }
    grp_sync(1);
    bk_arrive(sig0 + 8 * (ja % NSIG));
}

}  // namespace b200fft
