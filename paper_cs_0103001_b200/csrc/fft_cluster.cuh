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
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[pad16(lb + G::TPB * m)];
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

template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, bool ALIAS = false>
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
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k2 = la + G::TPA * m;
        const uint32_t owner = (uint32_t)(k2 / G::WB), line = (uint32_t)(k2 % G::WB);
        const uint32_t laddr = rx_s + (uint32_t)sizeof(Cx) * (line * G::LSB + pad16(n1));
        st_async_v2(mapa_u32(laddr, owner), v[FA::pos_out(m)], mapa_u32(bar_s, owner));
    }
    // ---- (B) rows k2 = c WB + tb, once all RX_BYTES have landed -------------
    mbar_wait_parity_cluster(bar_s, 0);
    const int tb = tid % G::WB, lb = tid / G::WB;
    const int k2 = c * G::WB + tb;
    Cx* lineb = rx + tb * G::LSB;
#pragma unroll
    for (int m = 0; m < E; ++m) v[FB::pos_in(m)] = lineb[pad16(lb + G::TPB * m)];
    FB::run(v, lineb, lb, twb);
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k1 = lb + G::TPB * m;
        dst[k2 + (int64_t)N2 * k1] = cscale(v[FB::pos_out(m)], scale);
    }
}

}  // namespace b200fft
