// fft_cluster.cuh -- one-HBM-pass large 1D FFT inside a thread-block cluster
// (sm_100a distributed shared memory).
//
// Computes, for every transform b of the batch, the paper's DFT (Eq. E2,
// PAPER.md P:78-80) X[k] = scale * sum_n x[n] W_N^{+-nk} with N = N1 * N2,
// by the four-step factorisation (an index split of the same sum):
//   n = n1 + N1 n2,  k = k2 + N2 k1
//   (A) Y[n1][k2] = sum_{n2} x[n1 + N1 n2] W_{N2}^{n2 k2}      column DFTs
//   (T) Y[n1][k2] *= W_N^{n1 k2}                               twiddle
//   (B) X[k2 + N2 k1] = sum_{n1} Y[n1][k2] W_{N1}^{n1 k1}      row DFTs
// One cluster of C CTAs owns one transform (512 KiB at N = 65536, more than
// one SM holds).  CTA c does the columns n1 in [c N1/C, (c+1) N1/C) of (A)
// and the rows k2 in [c N2/C, (c+1) N2/C) of (B); the transpose between
// them goes through DSMEM (each CTA stores straight into the owner's shared
// memory), so x is read from HBM once and X written once: 16 B/point.
//
// Lines are the thread-fastest index (consecutive threads = consecutive
// columns n1 in (A), consecutive rows k2 in (B)), so the global loads and
// stores are coalesced W-element runs and the smem exchanges stay
// conflict-free with odd line strides.
#pragma once
#include <cooperative_groups.h>

#include "fft_cols_pipe.cuh"
#include "fft_engine.cuh"

namespace b200fft {

__device__ __forceinline__ void cluster_arrive_release() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait_acquire() {
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <typename T, int N1, int N2, int C, int E>
struct ClusterCfg {
    static constexpr int WA = N1 / C;          // phase-A lines (columns n1) per CTA
    static constexpr int WB = N2 / C;          // phase-B lines (rows k2) per CTA
    static constexpr int TPA = N2 / E;         // threads per phase-A line
    static constexpr int TPB = N1 / E;         // threads per phase-B line
    static constexpr int NT = WA * TPA;        // threads per CTA
    static_assert(NT == WB * TPB, "phase A and B must use the same thread count");
    static constexpr int LSA = pad16c(N2) + 1;  // odd strides: lines are thread-fastest
    static constexpr int LSB = pad16c(N1) + 1;
    static constexpr int SMEM_ELEMS = (WA * LSA > WB * LSB) ? WA * LSA : WB * LSB;
    static constexpr size_t SMEM_BYTES = sizeof(cpx<T>) * SMEM_ELEMS;
};

// tw4: the four-step twiddles W_N^{n1 k2} laid out [k2][n1] (fp64-generated);
// twa / twb: the step tables of the N2- and N1-point in-CTA DFTs.
template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, int XMODE = 0>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(ClusterCfg<T, N1, N2, C, E>::NT, MINB)
    k_cluster(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t batch, T scale,
              const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb) {
    using Cx = cpx<T>;
    using G = ClusterCfg<T, N1, N2, C, E>;
    using FA = LineFFT<T, N2, E, INV>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* smem = reinterpret_cast<Cx*>(smem_raw);
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int c = (int)cluster.block_rank();
    const int64_t b = (int64_t)blockIdx.x / C;  // transform of this cluster
    const int tid = threadIdx.x;
    const Cx* src = in + b * N;
    Cx* dst = out + b * N;

    // ---- (A) columns n1 = c WA + t, elements n2 = la + TPA m ------------
    const int t = tid % G::WA, la = tid / G::WA;
    const int n1 = c * G::WA + t;
    Cx v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + G::TPA * m)];
    FA::run(v, smem + t * G::LSA, la, twa);
    // this CTA is done reading its smem for (A); the peers may overwrite it
    // once everyone has arrived (no ordering needed: the reads completed)
    // XMODE 1/2: timing experiments only (wrong results), see kernels_cluster.cu
    if constexpr (XMODE == 0 || XMODE == 2) cluster_arrive_relaxed();
    // ---- (T) twiddle W_N^{n1 k2}, k2 = la + TPA m (overlaps the barrier) --
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + G::TPA * m;
        v[FA::pos_out(m)] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
    }
    if constexpr (XMODE == 0 || XMODE == 2) cluster_wait_acquire();
    if constexpr (XMODE == 1 || XMODE == 2) __syncthreads();
    // ---- transpose through DSMEM: Y[n1][k2] -> owner of row k2 ------------
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + G::TPA * m;
        const int owner = k2 / G::WB, line = k2 % G::WB;
        if constexpr (XMODE == 1 || XMODE == 2) {
            smem[line * G::LSB + pad16(n1 % G::WA)] = v[FA::pos_out(m)];
        } else {
            Cx* remote = cluster.map_shared_rank(smem, owner);
            remote[line * G::LSB + pad16(n1)] = v[FA::pos_out(m)];
        }
    }
    // the stores above are visible to their owners after this barrier; after
    // it no CTA touches a peer's shared memory again (so no exit barrier)
    if constexpr (XMODE == 0 || XMODE == 2) {
        cluster_arrive_release();
        cluster_wait_acquire();
    } else {
        __syncthreads();
    }
    // ---- (B) rows k2 = c WB + tb, elements n1 = lb + TPB m -----------------
    const int tb = tid % G::WB, lb = tid / G::WB;
    const int k2 = c * G::WB + tb;
    Cx* lineb = smem + tb * G::LSB;
#pragma unroll
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[FB::bpos(lb, m)];
    FB::run(v, lineb, lb, twb);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k1 = lb + G::TPB * m;
        dst[k2 + (int64_t)N2 * k1] = cscale(v[FB::pos_out(m)], scale);
    }
}

// ---------------------------------------------------------------------------
// Variant 2 of the same computation: the transpose is pushed with
// st.async (asynchronous remote stores that complete_tx on the OWNER's
// mbarrier), into a receive buffer separate from the phase-A buffer.  No
// cluster-wide barrier sits between (A) and (B): each CTA waits only until
// its own mbarrier has counted all the bytes of its rows.  The single
// cluster barrier (publishing the mbarrier initialisation) is arrived at
// before phase (A) and waited on after it, so it costs nothing.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t mapa_u32(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, float2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];\n"
                 ::"r"(raddr), "f"(v.x), "f"(v.y), "r"(rbar) : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, double2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n"
                 ::"r"(raddr), "d"(v.x), "d"(v.y), "r"(rbar) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity_cluster(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar), "r"(parity) : "memory");
}

template <typename T, int N1, int N2, int C, int E, bool ALIAS = false>
struct Cluster2Cfg {
    using G = ClusterCfg<T, N1, N2, C, E>;
    static constexpr int A_ELEMS = G::WA * G::LSA;
    static constexpr int RX_ELEMS = G::WB * G::LSB;
    // ALIAS: the receive buffer is the phase-A buffer (half the smem; the
    // owner must have finished (A) before peers store -- one cluster barrier)
    static constexpr size_t RX_OFF = ALIAS ? 0 : sizeof(cpx<T>) * A_ELEMS;
    static constexpr size_t BAR_OFF =
        ALIAS ? sizeof(cpx<T>) * (A_ELEMS > RX_ELEMS ? A_ELEMS : RX_ELEMS) : RX_OFF + sizeof(cpx<T>) * RX_ELEMS;
    static constexpr size_t SMEM_BYTES = BAR_OFF + 16;
    static constexpr uint32_t RX_BYTES = (uint32_t)(sizeof(cpx<T>) * G::WB * N1);  // payload per CTA
};

// v[F::pos_out(m)] for a runtime m (a select chain; m is warp-uniform)
template <int M, int E, typename F, typename Cx>
__device__ __forceinline__ Cx pick_out(const Cx* v, int m) {
    if constexpr (M == E - 1) return v[F::pos_out(M)];
    else return (m == M) ? v[F::pos_out(M)] : pick_out<M + 1, E, F>(v, m);
}

template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, bool ALIAS = false, bool ROT = false>
__global__ void __cluster_dims__(C, 1, 1) __launch_bounds__(ClusterCfg<T, N1, N2, C, E>::NT, MINB)
    k_cluster2(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t batch, T scale,
               const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb) {
    using Cx = cpx<T>;
    using G = ClusterCfg<T, N1, N2, C, E>;
    using H = Cluster2Cfg<T, N1, N2, C, E, ALIAS>;
    using FA = LineFFT<T, N2, E, INV>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* bufa = reinterpret_cast<Cx*>(smem_raw);
    Cx* rx = reinterpret_cast<Cx*>(smem_raw + H::RX_OFF);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + H::BAR_OFF);
    const uint32_t bar_s = smem_u32(bar);
    namespace cg = cooperative_groups;
    const int c = (int)cg::this_cluster().block_rank();
    const int64_t b = (int64_t)blockIdx.x / C;
    const int tid = threadIdx.x;
    const Cx* src = in + b * N;
    Cx* dst = out + b * N;

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_s), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(H::RX_BYTES)
                     : "memory");
    }
    // publishes the initialised mbarrier (and, with ALIAS, "done with (A)")
    if constexpr (!ALIAS) cluster_arrive_relaxed();

    // ---- (A) columns n1 = c WA + t ----------------------------------------
    const int t = tid % G::WA, la = tid / G::WA;
    const int n1 = c * G::WA + t;
    Cx v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + G::TPA * m)];
    FA::run(v, bufa + t * G::LSA, la, twa);
    if constexpr (ALIAS) cluster_arrive_relaxed();
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + G::TPA * m;
        v[FA::pos_out(m)] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
    }
    cluster_wait_acquire();  // every peer's mbarrier is initialised
    // ---- transpose: st.async Y[n1][k2] into the owner's receive buffer ----
    const uint32_t rx_s = smem_u32(rx);
    if constexpr (ROT) {
        // rotate the send order by the CTA rank so that at every moment the
        // 16 CTAs of the cluster target 16 different owners (no incast)
#pragma unroll
        for (int mm = 0; mm < E; ++mm) {
            const int m = (mm + c) & (E - 1);
            const int k2 = la + G::TPA * m;
            const uint32_t owner = (uint32_t)(k2 / G::WB), line = (uint32_t)(k2 % G::WB);
            const uint32_t laddr = rx_s + (uint32_t)sizeof(Cx) * (line * G::LSB + pad16(n1));
            st_async_v2(mapa_u32(laddr, owner), pick_out<0, E, FA>(v, m), mapa_u32(bar_s, owner));
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k2 = la + G::TPA * m;
            const uint32_t owner = (uint32_t)(k2 / G::WB), line = (uint32_t)(k2 % G::WB);
            const uint32_t laddr = rx_s + (uint32_t)sizeof(Cx) * (line * G::LSB + pad16(n1));
            st_async_v2(mapa_u32(laddr, owner), v[FA::pos_out(m)], mapa_u32(bar_s, owner));
        }
    }
    // ---- (B) rows k2 = c WB + tb, once all RX_BYTES have landed -------------
    mbar_wait_parity_cluster(bar_s, 0);
    const int tb = tid % G::WB, lb = tid / G::WB;
    const int k2 = c * G::WB + tb;
    Cx* lineb = rx + tb * G::LSB;
#pragma unroll
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[FB::bpos(lb, m)];
    FB::run(v, lineb, lb, twb);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k1 = lb + G::TPB * m;
        dst[k2 + (int64_t)N2 * k1] = cscale(v[FB::pos_out(m)], scale);
    }
}

// ---------------------------------------------------------------------------
// Variant 3: the transpose as TMA bulk copies.  After (A) every CTA writes its
// outputs into its own smem grouped by owner (one 16 x 16 chunk per peer,
// XOR-swizzled so the owner reads it conflict-free), and 16 threads each issue
// one cp.async.bulk shared::cta -> shared::cluster copy of a whole chunk,
// completing on the owner's mbarrier.  Far fewer DSMEM transactions than one
// store per element.  Specialised to WA = WB = TPA = TPB = 16 (N1 = N2 = 256,
// C = 16, E = 16, 256 threads).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void bulk_s2s(uint32_t dst_cluster, uint32_t src_cta, uint32_t bytes,
                                         uint32_t bar_cluster) {
    asm volatile(
        "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            dst_cluster),
        "r"(src_cta), "r"(bytes), "r"(bar_cluster)
        : "memory");
}

template <typename T, int MINB, bool INV>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, MINB)
    k_cluster3(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t batch, T scale,
               const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb) {
    constexpr int N1 = 256, N2 = 256, C = 16, E = 16;
    using Cx = cpx<T>;
    using G = ClusterCfg<T, N1, N2, C, E>;
    static_assert(G::WA == 16 && G::WB == 16 && G::TPA == 16 && G::TPB == 16 && G::NT == 256, "shape");
    using FA = LineFFT<T, N2, E, INV>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    constexpr uint32_t CHUNK = 256 * sizeof(Cx);            // 16 x 16 elements per peer
    constexpr size_t A_BYTES = sizeof(Cx) * G::WA * G::LSA;  // >= 16 chunks
    static_assert(A_BYTES >= 16 * CHUNK, "send chunks must fit in the phase-A buffer");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    Cx* bufa = reinterpret_cast<Cx*>(smem_raw);
    Cx* rx = reinterpret_cast<Cx*>(smem_raw + A_BYTES);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + A_BYTES + 16 * CHUNK);
    const uint32_t bar_s = smem_u32(bar);
    namespace cg = cooperative_groups;
    const int c = (int)cg::this_cluster().block_rank();
    const int64_t b = (int64_t)blockIdx.x / C;
    const int tid = threadIdx.x;
    const Cx* src = in + b * N;
    Cx* dst = out + b * N;

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_s), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(16 * CHUNK)
                     : "memory");
    }
    cluster_arrive_relaxed();

    // ---- (A) columns n1 = 16 c + t, elements n2 = la + 16 m --------------
    const int t = tid & 15, la = tid >> 4;
    const int n1 = c * 16 + t;
    Cx v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + 16 * m)];
    FA::run(v, bufa + t * G::LSA, la, twa);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + 16 * m;
        v[FA::pos_out(m)] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
    }
    __syncthreads();  // every thread is done reading bufa
    // element k2 = la + 16 m belongs to owner m, row k2l = la: chunk m, swizzled
#pragma unroll
    for (int m = 0; m < E; ++m) bufa[m * 256 + la * 16 + (t ^ la)] = v[FA::pos_out(m)];
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncthreads();
    cluster_wait_acquire();  // every peer's mbarrier is initialised
    if (tid < 16) {
        const uint32_t q = (uint32_t)tid;
        const uint32_t dst_s = mapa_u32(smem_u32(rx) + (uint32_t)c * CHUNK, q);
        bulk_s2s(dst_s, smem_u32(bufa) + q * CHUNK, CHUNK, mapa_u32(bar_s, q));
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");  // bufa reusable
    }
    // ---- (B) rows k2 = 16 c + tb once the 16 chunks have landed -------------
    mbar_wait_parity_cluster(bar_s, 0);
    __syncthreads();  // the bulk reads of bufa are complete (tid < 16 waited)
    const int tb = tid & 15, lb = tid >> 4;
    const int k2 = c * 16 + tb;
#pragma unroll
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = rx[m * 256 + tb * 16 + (lb ^ tb)];
    Cx* lineb = bufa + tb * G::LSB;
    FB::run(v, lineb, lb, twb);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k1 = lb + 16 * m;
        dst[k2 + (int64_t)N2 * k1] = cscale(v[FB::pos_out(m)], scale);
    }
}

// ---------------------------------------------------------------------------
// The same four-step split as two cluster-free kernels that exchange through
// an L2-resident scratch (the batch is processed in chunks small enough that
// Y never leaves L2): k_step_a does (A)+(T) for WA columns and stores
// Y[k2][n1] (row k2 of Y = the input of (B)); k_step_b does (B) for WB rows.
// ---------------------------------------------------------------------------
template <typename T, int N1, int N2, int WA, int E, int MINB, bool INV>
__global__ void __launch_bounds__(WA*(N2 / E), MINB)
    k_step_a(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ y, const cpx<T>* __restrict__ tw4,
             const cpx<T>* __restrict__ twa) {
    using Cx = cpx<T>;
    using FA = LineFFT<T, N2, E, INV>;
    constexpr int TPA = N2 / E, LSA = pad16c(N2) + 1;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* smem = reinterpret_cast<Cx*>(smem_raw);
    const int64_t b = (int64_t)blockIdx.x / (N1 / WA);
    const int c = (int)(blockIdx.x % (N1 / WA));
    const int tid = threadIdx.x;
    const int t = tid % WA, la = tid / WA;
    const int n1 = c * WA + t;
    const Cx* src = in + b * N;
    Cx* dst = y + b * N;
    Cx v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + TPA * m)];
    FA::run(v, smem + t * LSA, la, twa);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + TPA * m;
        dst[(int64_t)k2 * N1 + n1] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
    }
}

template <typename T, int N1, int N2, int WB, int E, int MINB, bool INV>
__global__ void __launch_bounds__(WB*(N1 / E), MINB)
    k_step_b(const cpx<T>* __restrict__ y, cpx<T>* __restrict__ out, T scale, const cpx<T>* __restrict__ twb) {
    using Cx = cpx<T>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int TPB = N1 / E, LSB = pad16c(N1) + 1;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* smem = reinterpret_cast<Cx*>(smem_raw);
    const int64_t b = (int64_t)blockIdx.x / (N2 / WB);
    const int c = (int)(blockIdx.x % (N2 / WB));
    const int tid = threadIdx.x;
    // rows k2 are contiguous in y: lane-fastest mapping for coalesced loads
    const int tb = tid / TPB, lb = tid % TPB;
    const int k2 = c * WB + tb;
    const Cx* src = y + b * N + (int64_t)k2 * N1;
    Cx v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = src[lb + TPB * m];
    Cx* line = smem + tb * LSB;
    FB::run(v, line, lb, twb);
    // X[k2 + N2 k1]: stage through smem so that consecutive threads store
    // consecutive k2 (WB-element runs)
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) line[FB::bpos(lb, m)] = cscale(v[FB::pos_out(m)], scale);
    __syncthreads();
    Cx* dst = out + b * N + c * WB;
    for (int idx = tid; idx < WB * N1; idx += WB * TPB) {
        const int l = idx % WB, k1 = idx / WB;
        dst[(int64_t)N2 * k1 + l] = smem[l * LSB + pad16(k1)];
    }
}

// ---------------------------------------------------------------------------
// Variant 22: the two steps of one chunk pipelined across launches.  Launch i
// runs A(chunk i) and B(chunk i-1) side by side (disjoint CTAs): A writes Y
// into scratch slot i % 2, B reads slot (i-1) % 2.  Stream order makes A(i-1)
// complete before B(i-1) reads it and B(i-2) complete before A(i) overwrites
// its slot, so no events or flags are needed; every launch mixes HBM reads
// (A) with HBM writes (B), and Y stays in L2 (two slots of chunk x 512 KiB).
// Blocks [0, nA*16) are A tasks of transforms bA.., the rest B tasks.
// ---------------------------------------------------------------------------
template <typename T, int E, bool INV>
__global__ void __launch_bounds__(256, 4)
    k_step_ab(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, cpx<T>* __restrict__ ya,
              const cpx<T>* __restrict__ yb, int64_t bA, int nA, int64_t bB, T scale,
              const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb) {
    constexpr int N1 = 256, N2 = 256, W = 16;
    using Cx = cpx<T>;
    using F = LineFFT<T, 256, E, INV>;
    constexpr int TP = 256 / E, LS = pad16c(256) + 1;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* smem = reinterpret_cast<Cx*>(smem_raw);
    const int tid = threadIdx.x;
    const int blk = (int)blockIdx.x;
    if (blk < nA * 16) {
        const int64_t bl = blk / 16;
        const int c = blk % 16;
        const int t = tid % W, la = tid / W;
        const int n1 = c * W + t;
        const Cx* src = in + (bA + bl) * N;
        Cx* dst = ya + bl * N;
        Cx v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcs(src + n1 + (int64_t)N1 * (la + TP * m));
        F::run(v, smem + t * LS, la, twa);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k2 = la + TP * m;
            __stcg(dst + (int64_t)k2 * N1 + n1, cmul_dir<INV>(v[F::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1)));
        }
    } else {
        const int64_t bl = (blk - nA * 16) / 16;
        const int c = (blk - nA * 16) % 16;
        const int tb = tid / TP, lb = tid % TP;
        const int k2 = c * W + tb;
        const Cx* src = yb + bl * N + (int64_t)k2 * N1;
        Cx v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcg(src + lb + TP * m);
        Cx* line = smem + tb * LS;
        F::run(v, line, lb, twb);
        __syncthreads();
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lb, m)] = cscale(v[F::pos_out(m)], scale);
        __syncthreads();
        Cx* dst = out + (bB + bl) * N + c * W;
#pragma unroll
        for (int it = 0; it < (W * N1) / 256; ++it) {
            const int idx = tid + it * 256;
            const int l = idx % W, k1 = idx / W;
            __stcs(dst + (int64_t)N2 * k1 + l, smem[l * LS + pad16(k1)]);
        }
    }
}

// ---------------------------------------------------------------------------
// Persistent single-kernel form of the two steps: CTAs take tasks from a
// global ticket in the order A(0..Wr-1), B(0), A(Wr), B(1), A(Wr+1), ...,
// where A(b) / B(b) are the 16 column / 16 row tasks of transform b.  Y(b)
// lives in slot b mod Wr of a scratch ring small enough to stay in L2
// (Wr x 512 KiB), so HBM sees one read and one write per point.  B(b) waits
// for the 16 A(b) tasks (counter), A(b) waits for B(b - Wr) to free its slot.
// Every wait is on a task with a smaller ticket, held by a resident CTA
// (the grid is sized to the resident capacity), so the schedule cannot
// deadlock.  Streaming data uses evict-first loads/stores; Y uses .cg (L2).
// ---------------------------------------------------------------------------
struct FusedCtl {
    int* ticket;   // [1]
    int* done_a;   // [batch]
    int* done_b;   // [batch]
};

__device__ __forceinline__ void spin_until_geq(const int* p, int v) {
    int cur;
    while (true) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(cur) : "l"(p) : "memory");
        if (cur >= v) break;
        __nanosleep(64);
    }
}

template <typename T, int E, bool INV>
__global__ void __launch_bounds__(256, 4)
    k_fused_ab(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, cpx<T>* __restrict__ ring, int64_t batch,
               int wr, T scale, const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa,
               const cpx<T>* __restrict__ twb, FusedCtl ctl) {
    constexpr int N1 = 256, N2 = 256, W = 16, TP = 16, LS = pad16c(256) + 1;
    static_assert(E == 16, "256 threads = 16 lines x 16 threads");
    using Cx = cpx<T>;
    using F = LineFFT<T, 256, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* smem = reinterpret_cast<Cx*>(smem_raw);
    __shared__ int s_ticket;
    const int tid = threadIdx.x;
    const int64_t units = 2 * batch;
    const int64_t wq = batch < wr ? batch : wr;
    // dynamic tickets (measured faster than a static round-robin, which turns
    // CTA speed differences into dependency waits)
    while (true) {
        if (tid == 0) s_ticket = atomicAdd(ctl.ticket, 1);
        __syncthreads();
        const int64_t tk = s_ticket;
        __syncthreads();
        if (tk >= units * 16) break;
        const int64_t u = tk / 16;
        const int part = (int)(tk % 16);
        bool is_a;
        int64_t b;
        if (u < wq) {
            is_a = true;
            b = u;
        } else {
            const int64_t v = u - wq;
            if (v < 2 * (batch - wq)) {
                is_a = (v & 1) != 0;
                b = is_a ? v / 2 + wq : v / 2;
            } else {
                is_a = false;
                b = (batch - wq) + (v - 2 * (batch - wq));
            }
        }
        Cx* y = ring + (b % wr) * N;
        if (is_a) {
            if (b >= wr) {
                if (tid == 0) spin_until_geq(ctl.done_b + (b - wr), 16);
                __syncthreads();
            }
            const int t = tid % W, la = tid / W;
            const int n1 = part * W + t;
            const Cx* src = in + b * N;
            Cx v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcs(src + n1 + (int64_t)N1 * (la + TP * m));
            F::run(v, smem + t * LS, la, twa);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k2 = la + TP * m;
                __stcg(y + (int64_t)k2 * N1 + n1, cmul_dir<INV>(v[F::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1)));
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(ctl.done_a + b, 1);
        } else {
            if (tid == 0) spin_until_geq(ctl.done_a + b, 16);
            __syncthreads();
            const int tb = tid / TP, lb = tid % TP;
            const int k2 = part * W + tb;
            const Cx* src = y + (int64_t)k2 * N1;
            Cx v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcg(src + lb + TP * m);
            Cx* line = smem + tb * LS;
            F::run(v, line, lb, twb);
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m) line[F::bpos(lb, m)] = cscale(v[F::pos_out(m)], scale);
            __syncthreads();
            Cx* dst = out + b * N + part * W;
            for (int idx = tid; idx < W * N1; idx += 256) {
                const int l = idx % W, k1 = idx / W;
                __stcs(dst + (int64_t)N2 * k1 + l, smem[l * LS + pad16(k1)]);
            }
            __syncthreads();  // all reads of this Y slot are done before the release
            if (tid == 0) {
                __threadfence();
                atomicAdd(ctl.done_b + b, 1);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Variant 4: persistent, software-pipelined cluster kernel.  Each 16-CTA
// cluster loops over transforms; iteration i runs (A)+(T) of transform i,
// pushes it (st.async, rank-rotated) into slot i%2 of the owners' receive
// buffers, and only THEN runs (B) of transform i-1 -- so the DSMEM transfer
// of i overlaps the row work of i-1 instead of being waited for.
// Per slot: full[s] (owner side; 1 arrival = the owner's expect_tx + the
// peers' bytes) and empty[s] (sender side; 16 remote arrivals, one per owner
// that has consumed the slot).  Specialised to N1 = N2 = 256, C = 16, E = 16.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity_cta(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "W4_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W4_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

template <typename T>
struct Cluster4Cfg {
    using G = ClusterCfg<T, 256, 256, 16, 16>;
    static constexpr size_t A_BYTES = sizeof(cpx<T>) * G::WA * G::LSA;
    static constexpr size_t RX_BYTES_SLOT = sizeof(cpx<T>) * G::WB * G::LSB;
    static constexpr size_t BAR_OFF = A_BYTES + 2 * RX_BYTES_SLOT;
    static constexpr size_t SMEM_BYTES = BAR_OFF + 64;
    static constexpr uint32_t PAYLOAD = (uint32_t)(sizeof(cpx<T>) * 16 * 256);
};

template <typename T, int MINB, bool INV>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, MINB)
    k_cluster4(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t batch, T scale,
               const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb) {
    constexpr int N1 = 256, N2 = 256, E = 16;
    using Cx = cpx<T>;
    using G = ClusterCfg<T, N1, N2, 16, E>;
    using H = Cluster4Cfg<T>;
    using FA = LineFFT<T, N2, E, INV>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* bufa = reinterpret_cast<Cx*>(smem_raw);
    const uint32_t rx_s0 = smem_u32(smem_raw + H::A_BYTES);
    const uint32_t full0 = smem_u32(smem_raw + H::BAR_OFF);       // full[0], full[1]
    const uint32_t empty0 = full0 + 16;                            // empty[0], empty[1]
    namespace cg = cooperative_groups;
    const int c = (int)cg::this_cluster().block_rank();
    const int64_t cid = (int64_t)blockIdx.x / 16, ncl = (int64_t)gridDim.x / 16;
    const int tid = threadIdx.x;
    const int t = tid & 15, la = tid >> 4;  // phase A: line t (column), lane la
    const int n1 = c * 16 + t;
    const int64_t iters = (batch - cid + ncl - 1) / ncl;  // transforms of this cluster

    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(full0 + 8 * s), "r"(1) : "memory");
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(empty0 + 8 * s), "r"(16) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        for (int s = 0; s < 2; ++s)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(full0 + 8 * s),
                         "r"(H::PAYLOAD)
                         : "memory");
    }
    cluster_arrive_relaxed();
    bool cluster_synced = false;

    Cx v[E];
    auto phase_b = [&](int64_t j) {  // rows of transform j (iteration j of this cluster)
        const int s = (int)(j & 1);
        const uint32_t u = (uint32_t)(j >> 1);
        mbar_wait_parity_cta(full0 + 8 * s, u & 1);
        Cx* rx = reinterpret_cast<Cx*>(smem_raw + H::A_BYTES + s * H::RX_BYTES_SLOT);
        const int tb = tid & 15, lb = tid >> 4;
        Cx* lineb = rx + tb * G::LSB;
#pragma unroll
        for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[FB::bpos(lb, m)];
        FB::run(v, lineb, lb, twb);
        const int64_t b = cid + j * ncl;
        const int k2 = c * 16 + tb;
        Cx* dst = out + b * N;
#pragma unroll
        for (int m = 0; m < E; ++m) dst[k2 + (int64_t)N2 * (lb + 16 * m)] = cscale(v[FB::pos_out(m)], scale);
        __syncthreads();  // everyone is done with slot s
        if (j + 2 < iters) {
            if (tid == 0)  // re-arm this slot's next phase before releasing it
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(full0 + 8 * s),
                             "r"(H::PAYLOAD)
                             : "memory");
            __syncthreads();
            if (tid < 16) mbar_arrive_remote(mapa_u32(empty0 + 8 * s, (uint32_t)tid));
        }
    };

    for (int64_t i = 0; i < iters; ++i) {
        const int64_t b = cid + i * ncl;
        const Cx* src = in + b * N;
        // ---- (A) + (T) of transform i ----
#pragma unroll
        for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + 16 * m)];
        FA::run(v, bufa + t * G::LSA, la, twa);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k2 = la + 16 * m;
            v[FA::pos_out(m)] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
        }
        if (!cluster_synced) {
            cluster_wait_acquire();  // every peer's mbarriers are initialised
            cluster_synced = true;
        }
        // ---- push into slot i%2 of the owners, once they have freed it ----
        const int s = (int)(i & 1);
        const uint32_t u = (uint32_t)(i >> 1);
        if (u >= 1) mbar_wait_parity_cta(empty0 + 8 * s, (u - 1) & 1);
        const uint32_t rx_s = rx_s0 + (uint32_t)(s * H::RX_BYTES_SLOT);
#pragma unroll
        for (int mm = 0; mm < E; ++mm) {
            const int m = (mm + c) & (E - 1);
            const uint32_t owner = (uint32_t)m, line = (uint32_t)la;  // k2 = la + 16 m
            const uint32_t laddr = rx_s + (uint32_t)sizeof(Cx) * (line * G::LSB + pad16(n1));
            st_async_v2(mapa_u32(laddr, owner), pick_out<0, E, FA>(v, m), mapa_u32(full0 + 8 * s, owner));
        }
        __syncthreads();  // bufa is reused by the next (A); v is free
        // ---- (B) of the previous transform overlaps the transfer of this one ----
        if (i >= 1) phase_b(i - 1);
    }
    if (iters >= 1) phase_b(iters - 1);
    if (!cluster_synced) cluster_wait_acquire();
    // no CTA leaves while a peer may still signal or send to it
    cluster_arrive_release();
    cluster_wait_acquire();
}

// ---------------------------------------------------------------------------
// Variant 5: persistent 16-CTA clusters that exchange through an L2-resident
// per-cluster scratch slot (512 KiB, ~37 slots in flight) instead of DSMEM;
// cluster barriers order the slot's writes (A) and reads (B).  The second
// barrier (slot free again) is split: arrived after (B)'s loads, waited on
// just before the next (A) stores, so it overlaps (B)'s math and the next
// (A)'s loads and math.
// ---------------------------------------------------------------------------
template <typename T, int MINB, bool INV>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, MINB)
    k_cluster5(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, cpx<T>* __restrict__ scratch, int64_t batch,
               T scale, const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa,
               const cpx<T>* __restrict__ twb) {
    constexpr int N1 = 256, N2 = 256, E = 16, LS = pad16c(256) + 1;
    using Cx = cpx<T>;
    using F = LineFFT<T, 256, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* sm = reinterpret_cast<Cx*>(smem_raw);
    namespace cg = cooperative_groups;
    const int c = (int)cg::this_cluster().block_rank();
    const int64_t cid = (int64_t)blockIdx.x / 16, ncl = (int64_t)gridDim.x / 16;
    const int tid = threadIdx.x;
    Cx* y = scratch + cid * N;
    const int64_t iters = (batch - cid + ncl - 1) / ncl;
    for (int64_t j = 0; j < iters; ++j) {
        const int64_t b = cid + j * ncl;
        // ---- (A) + (T): columns n1 = 16 c + t -> Y[k2][n1] in the slot ----
        {
            const int t = tid & 15, la = tid >> 4;
            const int n1 = c * 16 + t;
            const Cx* src = in + b * N;
            Cx v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcs(src + n1 + (int64_t)N1 * (la + 16 * m));
            F::run(v, sm + t * LS, la, twa);
            if (j > 0) cluster_wait_acquire();  // the slot's previous readers are done
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k2 = la + 16 * m;
                __stcg(y + (int64_t)k2 * N1 + n1,
                       cmul_dir<INV>(v[F::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1)));
            }
        }
        cluster_arrive_release();
        cluster_wait_acquire();  // Y complete and visible
        // ---- (B): rows k2 = 16 c + tb, read lane-fastest (coalesced) ----
        {
            const int tb = tid >> 4, lb = tid & 15;
            const int k2 = c * 16 + tb;
            const Cx* src = y + (int64_t)k2 * N1;
            Cx v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[F::pos_in(m)] = __ldcg(src + lb + 16 * m);
            Cx* line = sm + tb * LS;
            F::run(v, line, lb, twb);
            // the loaded values have been consumed, so this CTA's reads of the
            // slot are complete: peers may overwrite it once all have arrived
            cluster_arrive_relaxed();
            __syncthreads();
#pragma unroll
            for (int m = 0; m < E; ++m) line[F::bpos(lb, m)] = cscale(v[F::pos_out(m)], scale);
            __syncthreads();
            Cx* dst = out + b * N + c * 16;
#pragma unroll
            for (int it = 0; it < 16; ++it) {
                const int idx = tid + it * 256;
                const int l = idx & 15, k1 = idx >> 4;
                __stcs(dst + (int64_t)N2 * k1 + l, sm[l * LS + pad16(k1)]);
            }
            __syncthreads();  // sm is reused by the next (A)
        }
    }
    if (iters > 0) cluster_wait_acquire();  // pair the last arrive before leaving
}

// ---------------------------------------------------------------------------
// Variant 6: variant 16 (st.async into the aliased phase-A buffer, rotated
// send order) made persistent -- one cluster loops over transforms
// cid, cid + ncl, ... -- and with the NEXT transform's phase-A columns
// prefetched into L2 (cp.async.bulk.prefetch, one 16-column row segment of
// 128 B per thread) while this one is transformed and exchanged, so the
// phase-A loads of every iteration after the first hit L2 and the HBM reads
// overlap the DSMEM exchange.  One cluster barrier per iteration (every CTA
// done with its phase-A smem before peers push into it), one mbarrier phase
// per iteration (parity i & 1).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

template <typename T, int MINB, bool INV, bool PREF>
__global__ void __cluster_dims__(16, 1, 1) __launch_bounds__(256, MINB)
    k_cluster6(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, int64_t batch, T scale,
               const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ twa, const cpx<T>* __restrict__ twb,
               unsigned stagger_ns) {
    constexpr int N1 = 256, N2 = 256, C = 16, E = 16;
    using Cx = cpx<T>;
    using G = ClusterCfg<T, N1, N2, C, E>;
    using H = Cluster2Cfg<T, N1, N2, C, E, true>;
    using FA = LineFFT<T, N2, E, INV>;
    using FB = LineFFT<T, N1, E, INV>;
    constexpr int64_t N = (int64_t)N1 * N2;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* bufa = reinterpret_cast<Cx*>(smem_raw);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + H::BAR_OFF);
    const uint32_t bar_s = smem_u32(bar);
    const uint32_t rx_s = smem_u32(bufa);
    namespace cg = cooperative_groups;
    const int c = (int)cg::this_cluster().block_rank();
    const int64_t cid = (int64_t)blockIdx.x / C, ncl = (int64_t)gridDim.x / C;
    const int tid = threadIdx.x;
    const int64_t iters = (batch - cid + ncl - 1) / ncl;
    const int t = tid % G::WA, la = tid / G::WA;
    const int n1 = c * G::WA + t;
    const int tb = tid % G::WB, lb = tid / G::WB;
    const int k2b = c * G::WB + tb;

    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar_s), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(H::RX_BYTES)
                     : "memory");
    }
    // staggered start: clusters resident on the same SMs begin a quarter
    // iteration apart so that their load / exchange / store phases interleave
    if (stagger_ns) {
        const unsigned d = (unsigned)(cid % 4) * stagger_ns;
        for (unsigned w = 0; w < d; w += 1000) __nanosleep(1000);
    }
    for (int64_t i = 0; i < iters; ++i) {
        const int64_t b = cid + i * ncl;
        const Cx* src = in + b * N;
        if constexpr (PREF) {
            if (i + 1 < iters)  // row n2 = tid of this CTA's 16 columns of the next transform
                prefetch_l2_bulk(src + ncl * N + (int64_t)N1 * tid + c * G::WA, (uint32_t)(G::WA * sizeof(Cx)));
        }
        // ---- (A) columns n1 = c WA + t ----
        Cx v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[FA::pos_in(m)] = src[n1 + (int64_t)N1 * (la + G::TPA * m)];
        FA::run(v, bufa + t * G::LSA, la, twa);
        // done with bufa (and, from the previous iteration, with rx = bufa)
        cluster_arrive_relaxed();
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k2 = la + G::TPA * m;
            v[FA::pos_out(m)] = cmul_dir<INV>(v[FA::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1));
        }
        cluster_wait_acquire();
#pragma unroll
        for (int mm = 0; mm < E; ++mm) {
            const int m = (mm + c) & (E - 1);
            const int k2 = la + G::TPA * m;
            const uint32_t owner = (uint32_t)(k2 / G::WB), line = (uint32_t)(k2 % G::WB);
            const uint32_t laddr = rx_s + (uint32_t)sizeof(Cx) * (line * G::LSB + pad16(n1));
            st_async_v2(mapa_u32(laddr, owner), pick_out<0, E, FA>(v, m), mapa_u32(bar_s, owner));
        }
        // ---- (B) rows k2 = c WB + tb, once all RX_BYTES have landed ----
        mbar_wait_parity_cluster(bar_s, (uint32_t)(i & 1));
        __syncthreads();  // every thread has observed phase i before it is re-armed
        if (tid == 0 && i + 1 < iters)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar_s), "r"(H::RX_BYTES)
                         : "memory");
        Cx* lineb = bufa + tb * G::LSB;
#pragma unroll
        for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[FB::bpos(lb, m)];
        FB::run(v, lineb, lb, twb);
        Cx* dst = out + b * N;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k1 = lb + G::TPB * m;
            dst[k2b + (int64_t)N2 * k1] = cscale(v[FB::pos_out(m)], scale);
        }
        __syncthreads();  // bufa is reused by the next (A)
    }
}

// ---------------------------------------------------------------------------
// Variant 28: the four-step split into independent 16-line tasks -- A(b, p):
// columns n1 in [16p, 16p+16) of transform b, (A)+(T), Y rows to an
// L2-resident ring slot; B(b, p): rows k2 in [16p, 16p+16) of Y(b), (B),
// X to HBM -- run by a persistent, software-pipelined grid.  Every CTA walks
// the global task sequence
//     A(0..D-1) | A(D) B(0) | A(D+1) B(1) | ... | B(batch-D..batch-1)
// (16 tasks per letter) with stride gridDim.x and prefetches its NEXT task's
// 16 x 256 input into the second smem stage with cp.async while it computes
// the current one, so HBM / L2 latency hides behind the math.  A B task's
// input waits on a counter (done_a[b] == 16) that was filled D transforms
// earlier in the sequence; an A task's ring slot waits on done_b of the
// transform RING slots back.  With 16 D >= gridDim.x every wait is on a
// task strictly earlier than the waiter's current one, so co-resident CTAs
// (cooperative launch) cannot deadlock.
// ---------------------------------------------------------------------------
struct AbCtl {
    int* done_a;  // [batch]
    int* done_b;  // [batch]
    int D, ring;
};

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <typename T, int MINB, bool INV>
__global__ void __launch_bounds__(256, MINB)
    k_ab_pipe(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out, cpx<T>* __restrict__ ring, int64_t batch,
              T scale, const cpx<T>* __restrict__ tw4, const cpx<T>* __restrict__ tw256, AbCtl ctl) {
    constexpr int N1 = 256, W = 16, E = 16, LS = pad16c(256) + 1;
    constexpr int64_t N = 65536;
    constexpr int STAGE = W * LS;
    using Cx = cpx<T>;
    using F = LineFFT<T, 256, E, INV>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    Cx* stage0 = reinterpret_cast<Cx*>(smem_raw);
    const int tid = threadIdx.x;
    const int t = tid % W, l = tid / W;  // line t (column n1 / row k2), lane l
    const int64_t Dp = batch < ctl.D ? batch : ctl.D;
    const int64_t n1t = 16 * Dp, n2t = 32 * (batch - Dp);
    const int64_t ntasks = 32 * batch;

    // task i -> (is_b, transform, part)
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
    // this thread's cp.async copies of a task's 16 x 256 tile into stage buf
    auto prefetch = [&](int64_t i, int buf) {
        if (i < ntasks) {
            bool isb;
            int64_t b;
            int part;
            decode(i, isb, b, part);
            Cx* sm = stage0 + buf * STAGE;
            if (!isb) {  // columns n1 = 16 part + tt, rows n2: 128-B runs
                const Cx* src = in + b * N + part * W;
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int idx = tid + it * 256;
                    const int tt = idx % W, r = idx / W;
                    cp_async8(sm + tt * LS + pad16(r), src + (int64_t)r * N1 + tt, true);
                }
            } else {  // rows k2 = 16 part + tt of Y (contiguous 2 KiB each)
                if (tid == 0) {
                    while (ld_acquire_gpu(ctl.done_a + b) < 16) __nanosleep(32);
                }
                __syncthreads();
                const Cx* src = ring + (b % ctl.ring) * N + (int64_t)part * W * N1;
#pragma unroll
                for (int it = 0; it < 16; ++it) {
                    const int idx = tid + it * 256;
                    const int tt = idx / N1, r = idx % N1;
                    cp_async8(sm + tt * LS + pad16(r), src + idx, true);
                }
            }
        }
        cp_async_commit();
    };

    int64_t i = blockIdx.x;
    prefetch(i, 0);
    for (int k = 0; i < ntasks; ++k, i += gridDim.x) {
        const int buf = k & 1;
        prefetch(i + gridDim.x, buf ^ 1);
        cp_async_wait<1>();
        __syncthreads();
        bool isb;
        int64_t b;
        int part;
        decode(i, isb, b, part);
        if (isb && tid == 0) {  // this task's reads of ring slot b are complete
            __threadfence();
            atomicAdd(ctl.done_b + b, 1);
        }
        Cx* line = stage0 + buf * STAGE + t * LS;
        Cx v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(l, m)];
        F::run(v, line, l, tw256);
        if (!isb) {
            const int n1 = part * W + t;
            if (b >= ctl.ring) {
                if (tid == 0) {
                    while (ld_acquire_gpu(ctl.done_b + (b - ctl.ring)) < 16) __nanosleep(32);
                }
                __syncthreads();
            }
            Cx* y = ring + (b % ctl.ring) * N;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k2 = l + 16 * m;
                __stcg(y + (int64_t)k2 * N1 + n1,
                       cmul_dir<INV>(v[F::pos_out(m)], __ldg(tw4 + (int64_t)k2 * N1 + n1)));
            }
            __threadfence();
            __syncthreads();
            if (tid == 0) atomicAdd(ctl.done_a + b, 1);
        } else {
            const int k2 = part * W + t;
            Cx* dst = out + b * N + k2;
#pragma unroll
            for (int m = 0; m < E; ++m) __stcs(dst + (int64_t)N1 * (l + 16 * m), cscale(v[F::pos_out(m)], scale));
            __syncthreads();  // stage buf is free for the prefetch two tasks ahead
        }
    }
    cp_async_wait<0>();
}

template <typename T>
constexpr size_t cluster3_smem() {
    using G = ClusterCfg<T, 256, 256, 16, 16>;
    return sizeof(cpx<T>) * G::WA * G::LSA + 16 * 256 * sizeof(cpx<T>) + 16;
}

}  // namespace b200fft
