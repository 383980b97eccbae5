// kernels_cluster.cu -- instantiations and launcher of the one-pass cluster
// FFT (fft_cluster.cuh) for 1D lengths that do not fit one CTA.
#include "fft_cluster.cuh"
#include "launch.h"

namespace b200fft {

namespace {

template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, int XMODE = 0>
cudaError_t cluster_t(const void* in, void* out, int64_t batch, double scale, const void* tw4,
                      const void* tw, cudaStream_t st) {
    using G = ClusterCfg<T, N1, N2, C, E>;
    auto kern = k_cluster<T, N1, N2, C, E, MINB, INV, XMODE>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM_BYTES);
        if (e == cudaSuccess && C > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (batch <= 0) return cudaSuccess;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(batch * C), G::NT, G::SMEM_BYTES, st>>>(
        reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out), batch, (T)scale,
        reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(N2), t + tw_base(N1));
    return cudaGetLastError();
}

template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, bool ALIAS = false>
cudaError_t cluster2_t(const void* in, void* out, int64_t batch, double scale, const void* tw4,
                       const void* tw, cudaStream_t st) {
    using G = ClusterCfg<T, N1, N2, C, E>;
    using H = Cluster2Cfg<T, N1, N2, C, E, ALIAS>;
    auto kern = k_cluster2<T, N1, N2, C, E, MINB, INV, ALIAS>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H::SMEM_BYTES);
        if (e == cudaSuccess && C > 8) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (batch <= 0) return cudaSuccess;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(batch * C), G::NT, H::SMEM_BYTES, st>>>(
        reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out), batch, (T)scale,
        reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(N2), t + tw_base(N1));
    return cudaGetLastError();
}

}  // namespace

bool cluster_supported(int prec, int64_t n, int* n1, int* n2) {
    if (prec != 0) return false;
    if (n == 65536) {
        *n1 = 256;
        *n2 = 256;
        return true;
    }
    return false;
}

template <bool INV>
cudaError_t cluster_65536(int variant, const void* in, void* out, int64_t batch, double scale, const void* tw4,
                          const void* tw, cudaStream_t st) {
    switch (variant) {
        case 0: return cluster_t<float, 256, 256, 16, 16, 4, INV>(in, out, batch, scale, tw4, tw, st);
        case 1: return cluster_t<float, 256, 256, 8, 32, 2, INV>(in, out, batch, scale, tw4, tw, st);
        case 2: return cluster_t<float, 256, 256, 16, 32, 4, INV>(in, out, batch, scale, tw4, tw, st);
        case 3: return cluster_t<float, 256, 256, 8, 16, 2, INV>(in, out, batch, scale, tw4, tw, st);
        case 4: return cluster2_t<float, 256, 256, 16, 16, 3, INV>(in, out, batch, scale, tw4, tw, st);
        case 5: return cluster2_t<float, 256, 256, 8, 32, 1, INV>(in, out, batch, scale, tw4, tw, st);
        case 6: return cluster2_t<float, 256, 256, 16, 32, 3, INV>(in, out, batch, scale, tw4, tw, st);
        // 8, 9: timing experiments only (WRONG results): the transpose stored
        // locally, without / with the two cluster barriers (C2 notes)
        case 8: return cluster_t<float, 256, 256, 16, 16, 4, INV, 1>(in, out, batch, scale, tw4, tw, st);
        case 9: return cluster_t<float, 256, 256, 16, 16, 4, INV, 2>(in, out, batch, scale, tw4, tw, st);
        case 7: return cluster2_t<float, 256, 256, 8, 16, 1, INV>(in, out, batch, scale, tw4, tw, st);
        case 10: return cluster2_t<float, 256, 256, 16, 16, 4, INV, true>(in, out, batch, scale, tw4, tw, st);
        case 11: return cluster2_t<float, 256, 256, 8, 32, 2, INV, true>(in, out, batch, scale, tw4, tw, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_cluster(int prec, bool inv, int64_t n, const void* in, void* out, int64_t batch,
                           double scale, const void* tw4, const void* tw, int variant, cudaStream_t st) {
    if (prec == 0 && n == 65536)
        return inv ? cluster_65536<true>(variant, in, out, batch, scale, tw4, tw, st)
                   : cluster_65536<false>(variant, in, out, batch, scale, tw4, tw, st);
    return cudaErrorInvalidValue;
}

}  // namespace b200fft
