// kernels_cluster.cu -- instantiations and launcher of the one-pass cluster
// FFT (fft_cluster.cuh) for 1D lengths that do not fit one CTA.
#include <cudaTypedefs.h>

#include <cstdio>

#include "fft_abbulk.cuh"
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

template <typename T, int N1, int N2, int C, int E, int MINB, bool INV, bool ALIAS = false, bool ROT = false>
cudaError_t cluster2_t(const void* in, void* out, int64_t batch, double scale, const void* tw4,
                       const void* tw, cudaStream_t st) {
    using G = ClusterCfg<T, N1, N2, C, E>;
    using H = Cluster2Cfg<T, N1, N2, C, E, ALIAS>;
    auto kern = k_cluster2<T, N1, N2, C, E, MINB, INV, ALIAS, ROT>;
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

template <typename T, int MINB, bool INV>
cudaError_t cluster3_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    constexpr size_t smem = cluster3_smem<T>();
    auto kern = k_cluster3<T, MINB, INV>;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (batch <= 0) return cudaSuccess;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(batch * 16), 256, smem, st>>>(reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out),
                                                   batch, (T)scale, reinterpret_cast<const cpx<T>*>(tw4),
                                                   t + tw_base(256), t + tw_base(256));
    return cudaGetLastError();
}

// two cluster-free kernels per chunk of transforms; Y stays in L2 between them
template <typename T, int WA, int WB, int E, int MINB, bool INV>
cudaError_t step_ab_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                      cudaStream_t st) {
    constexpr int N1 = 256, N2 = 256;
    constexpr size_t smem_a = sizeof(cpx<T>) * WA * (pad16c(N2) + 1);
    constexpr size_t smem_b = sizeof(cpx<T>) * WB * (pad16c(N1) + 1);
    auto ka = k_step_a<T, N1, N2, WA, E, MINB, INV>;
    auto kb = k_step_b<T, N1, N2, WB, E, MINB, INV>;
    static bool attr = false;
    static void* scratch = nullptr;
    static int64_t chunk = 0;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(ka, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_a);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_b);
        const char* cs = getenv("B200FFT_STEP_CHUNK");
        chunk = cs ? atoll(cs) : 64;
        if (e == cudaSuccess) e = cudaMalloc(&scratch, (size_t)chunk * N1 * N2 * sizeof(cpx<T>));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    const cpx<T>* x = reinterpret_cast<const cpx<T>*>(in);
    cpx<T>* o = reinterpret_cast<cpx<T>*>(out);
    cpx<T>* y = reinterpret_cast<cpx<T>*>(scratch);
    for (int64_t b0 = 0; b0 < batch; b0 += chunk) {
        const int64_t nb = batch - b0 < chunk ? batch - b0 : chunk;
        ka<<<(unsigned)(nb * (N1 / WA)), WA * (N2 / E), smem_a, st>>>(x + b0 * N1 * N2, y,
                                                                    reinterpret_cast<const cpx<T>*>(tw4),
                                                                    t + tw_base(N2));
        kb<<<(unsigned)(nb * (N2 / WB)), WB * (N1 / E), smem_b, st>>>(y, o + b0 * N1 * N2, (T)scale, t + tw_base(N1));
    }
    return cudaGetLastError();
}

template <typename T, bool INV>
cudaError_t fused_ab_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    constexpr size_t smem = sizeof(cpx<T>) * 16 * (pad16c(256) + 1);
    auto k = k_fused_ab<T, 16, INV>;
    static bool attr = false;
    static void* ring = nullptr;
    static int* ctl = nullptr;
    static int64_t ctl_n = 0;
    static int wr = 0, grid = 0;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const char* rs = getenv("B200FFT_RING");
        wr = rs ? atoi(rs) : 32;
        if (e == cudaSuccess) e = cudaMalloc(&ring, (size_t)wr * 65536 * sizeof(cpx<T>));
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
        if (e != cudaSuccess) return e;
        grid = sms * occ;
        attr = true;
    }
    if (batch <= 0) return cudaSuccess;
    if (ctl_n < 1 + 2 * batch) {
        if (ctl) cudaFree(ctl);
        cudaError_t e = cudaMalloc(&ctl, sizeof(int) * (1 + 2 * batch));
        if (e != cudaSuccess) return e;
        ctl_n = 1 + 2 * batch;
    }
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(int) * (1 + 2 * batch), st);
    if (e != cudaSuccess) return e;
    FusedCtl c{ctl, ctl + 1, ctl + 1 + batch};
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    const int64_t tasks = 32 * batch;
    const int g = (int)(tasks < grid ? tasks : grid);
    k<<<g, 256, smem, st>>>(reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out),
                            reinterpret_cast<cpx<T>*>(ring), batch, wr, (T)scale,
                            reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(256), t + tw_base(256), c);
    return cudaGetLastError();
}

template <typename T, int MINB, bool INV>
cudaError_t cluster4_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    using H = Cluster4Cfg<T>;
    auto kern = k_cluster4<T, MINB, INV>;
    static int max_clusters = 0;
    if (!max_clusters) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H::SMEM_BYTES);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(16 * 64, 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = H::SMEM_BYTES;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess) return e;
        max_clusters = n > 0 ? n : 1;
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t ncl = batch < max_clusters ? batch : max_clusters;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(ncl * 16), 256, H::SMEM_BYTES, st>>>(reinterpret_cast<const cpx<T>*>(in),
                                                          reinterpret_cast<cpx<T>*>(out), batch, (T)scale,
                                                          reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(256),
                                                          t + tw_base(256));
    return cudaGetLastError();
}

template <typename T, int MINB, bool INV>
cudaError_t cluster5_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    constexpr size_t smem = sizeof(cpx<T>) * 16 * (pad16c(256) + 1);
    auto kern = k_cluster5<T, MINB, INV>;
    static int max_clusters = 0;
    static void* scratch = nullptr;
    if (!max_clusters) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(16 * 64, 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e == cudaSuccess) e = cudaMalloc(&scratch, (size_t)(n > 0 ? n : 1) * 65536 * sizeof(cpx<T>));
        if (e != cudaSuccess) return e;
        max_clusters = n > 0 ? n : 1;
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t ncl = batch < max_clusters ? batch : max_clusters;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(ncl * 16), 256, smem, st>>>(reinterpret_cast<const cpx<T>*>(in), reinterpret_cast<cpx<T>*>(out),
                                                 reinterpret_cast<cpx<T>*>(scratch), batch, (T)scale,
                                                 reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(256),
                                                 t + tw_base(256));
    return cudaGetLastError();
}

template <typename T, int MINB, bool INV, bool PREF>
cudaError_t cluster6_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    using H = Cluster2Cfg<T, 256, 256, 16, 16, true>;
    auto kern = k_cluster6<T, MINB, INV, PREF>;
    static int max_clusters = 0;
    static unsigned stagger = 0;
    if (!max_clusters) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)H::SMEM_BYTES);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 16;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(16 * 64, 1, 1);
        cfg.blockDim = dim3(256, 1, 1);
        cfg.dynamicSmemBytes = H::SMEM_BYTES;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
        if (e != cudaSuccess) return e;
        const char* f = getenv("B200FFT_CLUSTERS");
        if (f && atoi(f) > 0 && atoi(f) < n) n = atoi(f);
        max_clusters = n > 0 ? n : 1;
        const char* sg = getenv("B200FFT_STAGGER_NS");
        stagger = sg ? (unsigned)atoi(sg) : 0u;
        fprintf(stderr, "cluster6: max active clusters %d, stagger %u ns\n", max_clusters, stagger);
    }
    if (batch <= 0) return cudaSuccess;
    const int64_t ncl = batch < max_clusters ? batch : max_clusters;
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    kern<<<(unsigned)(ncl * 16), 256, H::SMEM_BYTES, st>>>(reinterpret_cast<const cpx<T>*>(in),
                                                          reinterpret_cast<cpx<T>*>(out), batch, (T)scale,
                                                          reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(256),
                                                          t + tw_base(256), stagger);
    return cudaGetLastError();
}

template <typename T, bool INV>
cudaError_t step_ab2_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                       cudaStream_t st) {
    constexpr size_t smem = sizeof(cpx<T>) * 16 * (pad16c(256) + 1);
    auto k = k_step_ab<T, 16, INV>;
    static bool attr = false;
    static void* scratch = nullptr;
    static int64_t chunk = 0;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        const char* cs = getenv("B200FFT_STEP_CHUNK");
        chunk = cs ? atoll(cs) : 48;
        if (e == cudaSuccess) e = cudaMalloc(&scratch, (size_t)2 * chunk * 65536 * sizeof(cpx<T>));
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    const cpx<T>* x = reinterpret_cast<const cpx<T>*>(in);
    cpx<T>* o = reinterpret_cast<cpx<T>*>(out);
    cpx<T>* y = reinterpret_cast<cpx<T>*>(scratch);
    const int64_t nch = (batch + chunk - 1) / chunk;
    for (int64_t i = 0; i <= nch; ++i) {
        const int64_t bA = i * chunk, bB = (i - 1) * chunk;
        const int nA = i < nch ? (int)(batch - bA < chunk ? batch - bA : chunk) : 0;
        const int nB = i >= 1 ? (int)(batch - bB < chunk ? batch - bB : chunk) : 0;
        cpx<T>* ya = y + (i & 1) * chunk * 65536;
        const cpx<T>* yb = y + ((i + 1) & 1) * chunk * 65536;
        k<<<(unsigned)(16 * (nA + nB)), 256, smem, st>>>(x, o, ya, yb, bA, nA, bB, (T)scale,
                                                        reinterpret_cast<const cpx<T>*>(tw4), t + tw_base(256),
                                                        t + tw_base(256));
    }
    return cudaGetLastError();
}

template <typename T, int MINB, bool INV>
cudaError_t ab_pipe_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                      cudaStream_t st) {
    constexpr size_t smem = 2 * sizeof(cpx<T>) * 16 * (pad16c(256) + 1);
    auto k = k_ab_pipe<T, MINB, INV>;
    static int grid = 0, D = 0, ring_slots = 0;
    static void* ring = nullptr;
    static int* ctl = nullptr;
    static int64_t ctl_n = 0;
    if (!grid) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, smem);
        if (e != cudaSuccess) return e;
        grid = sms * (occ > 0 ? occ : 1);
        const char* dv = getenv("B200FFT_AB_D");
        D = (grid + 15) / 16 + (dv ? atoi(dv) : 8);
        const char* rv = getenv("B200FFT_AB_RING");
        ring_slots = D + (rv ? atoi(rv) : 16);
        e = cudaMalloc(&ring, (size_t)ring_slots * 65536 * sizeof(cpx<T>));
        if (e != cudaSuccess) return e;
        fprintf(stderr, "ab_pipe: grid %d (occ %d), D %d, ring %d\n", grid, occ, D, ring_slots);
    }
    if (batch <= 0) return cudaSuccess;
    if (ctl_n < 2 * batch) {
        if (ctl) cudaFree(ctl);
        cudaError_t e = cudaMalloc(&ctl, sizeof(int) * 2 * batch);
        if (e != cudaSuccess) return e;
        ctl_n = 2 * batch;
    }
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(int) * 2 * batch, st);
    if (e != cudaSuccess) return e;
    AbCtl c{ctl, ctl + batch, D, ring_slots};
    const cpx<T>* t = reinterpret_cast<const cpx<T>*>(tw);
    const int64_t tasks = 32 * batch;
    const int g = (int)(tasks < grid ? tasks : grid);
    const cpx<T>* a_in = reinterpret_cast<const cpx<T>*>(in);
    cpx<T>* a_out = reinterpret_cast<cpx<T>*>(out);
    cpx<T>* a_ring = reinterpret_cast<cpx<T>*>(ring);
    T a_scale = (T)scale;
    const cpx<T>* a_tw4 = reinterpret_cast<const cpx<T>*>(tw4);
    const cpx<T>* a_tw = t + tw_base(256);
    void* args[] = {&a_in, &a_out, &a_ring, &batch, &a_scale, &a_tw4, &a_tw, &c};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3(g, 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, (const void*)k, args);
}

template <bool INV>
cudaError_t ab_bulk_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                      cudaStream_t st) {
    using G = AbBulkCfg;
    auto k = k_ab_bulk<INV>;
    static int grid = 0, D = 0, ring_slots = 0;
    static void* ring = nullptr;
    static int* ctl = nullptr;
    static int64_t ctl_n = 0;
    if (!grid) {
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 256, G::SMEM);
        if (e != cudaSuccess) return e;
        grid = sms * (occ > 0 ? occ : 1);
        D = (2 * grid + 15) / 16 + 8;
        const char* rv = getenv("B200FFT_AB_RING");
        ring_slots = D + (rv ? atoi(rv) : 16);
        e = cudaMalloc(&ring, (size_t)ring_slots * 65536 * sizeof(float2));
        if (e != cudaSuccess) return e;
        if (getenv("B200FFT_VERBOSE")) fprintf(stderr, "ab_bulk: grid %d (occ %d), D %d, ring %d\n", grid, occ, D, ring_slots);
    }
    if (batch <= 0) return cudaSuccess;
    if (ctl_n < 2 * batch) {
        if (ctl) cudaFree(ctl);
        cudaError_t e = cudaMalloc(&ctl, sizeof(int) * 2 * batch);
        if (e != cudaSuccess) return e;
        ctl_n = 2 * batch;
    }
    cudaError_t e = cudaMemsetAsync(ctl, 0, sizeof(int) * 2 * batch, st);
    if (e != cudaSuccess) return e;
    AbBulkCtl c{ctl, ctl + batch, D, ring_slots};
    const float2* a_in = reinterpret_cast<const float2*>(in);
    float2* a_out = reinterpret_cast<float2*>(out);
    float2* a_ring = reinterpret_cast<float2*>(ring);
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256);
    int64_t a_batch = batch;
    void* args[] = {&a_in, &a_out, &a_ring, &a_batch, &a_scale, &a_tw4, &a_tw, &c};
    const int64_t tasks = 32 * batch;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)(tasks < grid ? tasks : grid), 1, 1);
    cfg.blockDim = dim3(256, 1, 1);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, (const void*)k, args);
}

// tensor maps of variant 41 (cuTensorMapEncodeTiled through the runtime's
// driver entry point: no libcuda link)
bool encode3(CUtensorMap* map, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
             int swz) {  // swz: 0, 64 or 128 (B TMA swizzle span)
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !enc)
            return false;
    }
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
    const cuuint32_t box[3] = {b0, b1, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : (swz == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE), CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// launch geometry of variants 41 / 42 (cached per kernel): persistent grid,
// dependency distance D (transforms) and ring slots
struct AbGeom {
    int grid = 0, D = 0, ring = 0;
};
template <bool INV, bool WS, int NSV = 3>
cudaError_t ab_geom(AbGeom* g) {
    static AbGeom cached;
    if (!cached.grid) {
        constexpr size_t SMEM = WS ? AbWsCfgN<NSV>::SMEM : AbTmaCfg::SMEM;
        constexpr int NT = WS ? 288 : 256;
        auto k = WS ? k_ab_ws<INV, NSV> : k_ab_tma<INV>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NT, SMEM);
        if (e != cudaSuccess) return e;
        AbGeom t;
        t.grid = sms * (occ > 0 ? occ : 1);
        const char* gv = getenv("B200FFT_AB_GRID");
        if (gv && atoi(gv) > 0 && atoi(gv) < t.grid) t.grid = atoi(gv);
        // every wait must point at least (tasks in flight per CTA) x grid
        // positions back in the task order: 2 for 41, NS = 3 for 42
        const int depth = WS ? NSV : 2;
        const char* dv = getenv("B200FFT_AB_D");
        t.D = (depth * t.grid + 15) / 16 + (dv ? atoi(dv) : 8);
        const char* rv = getenv("B200FFT_AB_RING");
        // ring = D + 24 slots: an A store waits on the B parts 24 transforms
        // (768 task positions) back, always an earlier task; 24 measured best
        // for variant 44 (B200FFT_AB_RING sweeps it)
        t.ring = t.D + (rv ? atoi(rv) : 24);
        if (getenv("B200FFT_VERBOSE"))
            fprintf(stderr, "ab_tma(ws=%d): grid %d (occ %d), D %d, ring %d\n", (int)WS, t.grid, occ, t.D, t.ring);
        cached = t;
    }
    *g = cached;
    return cudaSuccess;
}

// variants 45 / 46 (8-line tasks, 32 parts per phase)
template <bool INV, int NS, int MINB>
cudaError_t ab8_geom(AbGeom* g) {
    static AbGeom cached;
    if (!cached.grid) {
        constexpr size_t SMEM = AbWs8Cfg<NS>::SMEM;
        auto k = k_ab_ws8<INV, NS, MINB>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 288, SMEM);
        if (e != cudaSuccess) return e;
        AbGeom t;
        t.grid = sms * (occ > 0 ? occ : 1);
        const char* gv = getenv("B200FFT_AB_GRID");
        if (gv && atoi(gv) > 0 && atoi(gv) < t.grid) t.grid = atoi(gv);
        // waits point at least NS x grid task positions back (32 per transform)
        const char* dv = getenv("B200FFT_AB_D");
        t.D = (NS * t.grid + 31) / 32 + (dv ? atoi(dv) : 8);
        const char* rv = getenv("B200FFT_AB_RING");
        t.ring = t.D + (rv ? atoi(rv) : 24);
        if (getenv("B200FFT_VERBOSE"))
            fprintf(stderr, "ab_ws8<%d,%d>: grid %d (occ %d), D %d, ring %d\n", NS, MINB, t.grid, occ, t.D, t.ring);
        cached = t;
    }
    *g = cached;
    return cudaSuccess;
}

// caller-provided scratch: the Y ring (ring x 512 KiB) then the counters
size_t ab_ws_bytes(int64_t ring, int64_t batch) {
    return (size_t)ring * 65536 * sizeof(float2) + (size_t)2 * batch * sizeof(int);
}

// Grid of one task-pipeline launch.  A CTA's A task at local index k is
// signalled (done_a) only once its producer has issued its loads up to local
// index k + NS - 1 (or its last one), i.e. task position j + (NS - 1) grid.
// A B load at position i waits for A parts at positions j <= i - d, so the
// schedule is deadlock-free when every such distance d exceeds (NS - 1) grid:
// in the steady state d >= 16 D + 1 (D is sized for it, ab_geom); with fewer
// transforms than D every A precedes every B and d >= PP (batch - 1) + 1,
// so the grid is capped there -- unless every CTA holds at most one task.
int64_t ab_launch_grid(int64_t grid, int64_t batch, int64_t D, int PP, int NS) {
    const int64_t tasks = 2 * (int64_t)PP * batch;
    if (tasks <= grid) return tasks;
    if (batch >= D || NS <= 1 || getenv("B200FFT_AB_NOCAP")) return grid;
    const int64_t cap = ((int64_t)PP * (batch - 1)) / (NS - 1);  // (NS - 1) g <= PP (batch - 1) < d
    return cap < 1 ? 1 : (cap < grid ? cap : grid);
}

template <bool INV, bool WS = false, int NSV = 3>
cudaError_t ab_tma_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                     void* ws, size_t ws_bytes, cudaStream_t st) {
    constexpr size_t SMEM = WS ? AbWsCfgN<NSV>::SMEM : AbTmaCfg::SMEM;
    constexpr int NT = WS ? 288 : 256;
    auto k = WS ? k_ab_ws<INV, NSV> : k_ab_tma<INV>;
    AbGeom g;
    cudaError_t e = ab_geom<INV, WS, NSV>(&g);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    if (!ws || ws_bytes < ab_ws_bytes(g.ring, batch)) return cudaErrorInvalidValue;
    void* ring = ws;
    int* ctl = reinterpret_cast<int*>((char*)ws + (size_t)g.ring * 65536 * sizeof(float2));
    CUtensorMap m_x, m_out, m_yst, m_yld;
    if (!encode3(&m_x, const_cast<void*>(in), 256, 256, (uint64_t)batch, 16, 256, 0) ||
        !encode3(&m_out, out, 256, 256, (uint64_t)batch, 16, 256, 128) ||
        !encode3(&m_yst, ring, 256, 256, g.ring, 16, 256, 0) ||
        !encode3(&m_yld, ring, 256, 256, g.ring, 256, 16, 0))
        return cudaErrorInvalidValue;
    e = cudaMemsetAsync(ctl, 0, sizeof(int) * 2 * batch, st);
    if (e != cudaSuccess) return e;
    AbBulkCtl c{ctl, ctl + batch, g.D, g.ring};
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256);
    int64_t a_batch = batch;
    const float2* a_ring = reinterpret_cast<const float2*>(ring);
    static const int opts = [] {
        const char* v = getenv("B200FFT_AB_OPTS");
        // bits: 1 / 4 discard consumed Y rows from L2 (producer / compute
        // warps: fewer DRAM writes, not faster), 2 / 8 signal orders, 16 x d:
        // L2 tensor prefetch of the A tile d tasks ahead (d = 1 measured best)
        // 128: the A twiddles W_N^{n1 k2} by a 15-step product from two table
        // entries instead of 16 loads (-4.5%)
        const int o = v ? atoi(v) : 144;
        // 512: drop the A -> B and ring waits (timing experiment, wrong results)
        return (o & 512) && !getenv("B200FFT_ALLOW_WRONG") ? (o & ~512) : o;
    }();
    int a_opts = opts;
    void* args[] = {&m_x, &m_yst, &m_yld, &m_out, &a_batch, &a_scale, &a_tw4, &a_tw, &c, &a_ring, &a_opts};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)ab_launch_grid(g.grid, batch, g.D, 16, WS ? NSV : 2), 1, 1);
    cfg.blockDim = dim3(NT, 1, 1);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // An L2 access-policy window marks the Y ring persisting for this launch
    // (with a device persisting-L2 set-aside of the ring's size, set once):
    // the ring then never spills to HBM (ncu: DRAM bytes = algorithmic,
    // 1.10 -> 1.07 ms).  B200FFT_AB_PERSIST=0 turns it off.
    static const bool persist = [] {
        const char* v = getenv("B200FFT_AB_PERSIST");
        return !(v && v[0] == '0');
    }();
    if (persist) {
        static bool limit_set = false;
        const size_t rb = (size_t)g.ring * 65536 * sizeof(float2);
        if (!limit_set) {
            int dev = 0, mx = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
            // B200FFT_AB_PERSIST_FRAC: set-aside as a fraction of the ring (1 = all of it)
            const char* fv = getenv("B200FFT_AB_PERSIST_FRAC");
            const double fr = fv ? atof(fv) : 1.0;
            const size_t want = (size_t)((double)rb * (fr > 0 ? fr : 1.0));
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want < (size_t)mx ? want : (size_t)mx);
            if (getenv("B200FFT_VERBOSE")) fprintf(stderr, "persisting L2 max %d, ring %zu\n", mx, rb);
            limit_set = true;
        }
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = ring;
        attr[1].val.accessPolicyWindow.num_bytes = rb;
        static const float hit = [] {
            const char* hv = getenv("B200FFT_AB_HIT");
            return hv ? (float)atof(hv) : 1.0f;
        }();
        attr[1].val.accessPolicyWindow.hitRatio = hit;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelExC(&cfg, (const void*)k, args);
}

// variant 47 (direct Y stores, fft_abbulk.cuh k_ab_ds)
template <bool INV>
cudaError_t ds_geom(AbGeom* g) {
    static AbGeom cached;
    if (!cached.grid) {
        constexpr size_t SMEM = AbDsCfg::SMEM;
        auto k = k_ab_ds<INV>;
        cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        int dev = 0, sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaGetDevice(&dev);
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 288, SMEM);
        if (e != cudaSuccess) return e;
        AbGeom t;
        t.grid = sms * (occ > 0 ? occ : 1);
        // done_a is released one load later than in 44: waits must point
        // (NS = 2) x grid positions back, plus margin
        const char* dv = getenv("B200FFT_AB_D");
        t.D = (3 * t.grid + 15) / 16 + (dv ? atoi(dv) : 8);
        const char* rv = getenv("B200FFT_AB_RING");
        t.ring = t.D + (rv ? atoi(rv) : 24);
        if (getenv("B200FFT_VERBOSE"))
            fprintf(stderr, "ab_ds: grid %d (occ %d), D %d, ring %d\n", t.grid, occ, t.D, t.ring);
        cached = t;
    }
    *g = cached;
    return cudaSuccess;
}

template <bool INV>
cudaError_t ab_ds_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
    auto k = k_ab_ds<INV>;
    AbGeom g;
    cudaError_t e = ds_geom<INV>(&g);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    if (!ws || ws_bytes < ab_ws_bytes(g.ring, batch)) return cudaErrorInvalidValue;
    void* ring = ws;
    int* ctl = reinterpret_cast<int*>((char*)ws + (size_t)g.ring * 65536 * sizeof(float2));
    CUtensorMap m_x, m_out, m_yst, m_yld;
    if (!encode3(&m_x, const_cast<void*>(in), 256, 256, (uint64_t)batch, 16, 256, 0) ||
        !encode3(&m_out, out, 256, 256, (uint64_t)batch, 16, 256, 128) ||
        !encode3(&m_yst, ring, 256, 256, g.ring, 16, 256, 0) || !encode3(&m_yld, ring, 256, 256, g.ring, 256, 16, 0))
        return cudaErrorInvalidValue;
    e = cudaMemsetAsync(ctl, 0, sizeof(int) * 2 * batch, st);
    if (e != cudaSuccess) return e;
    AbBulkCtl c{ctl, ctl + batch, g.D, g.ring};
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256);
    int64_t a_batch = batch;
    const float2* a_ring = reinterpret_cast<const float2*>(ring);
    static const int opts = [] {
        const char* v = getenv("B200FFT_AB_OPTS");
        return v ? atoi(v) : 16;
    }();
    int a_opts = opts;
    void* args[] = {&m_x, &m_yst, &m_yld, &m_out, &a_batch, &a_scale, &a_tw4, &a_tw, &c, &a_ring, &a_opts};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)ab_launch_grid(g.grid, batch, g.D, 16, 3), 1, 1);
    cfg.blockDim = dim3(288, 1, 1);
    cfg.dynamicSmemBytes = AbDsCfg::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static bool limit_set = false;
    const size_t rb = (size_t)g.ring * 65536 * sizeof(float2);
    if (!limit_set) {
        int dev = 0, mx = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, rb < (size_t)mx ? rb : (size_t)mx);
        limit_set = true;
    }
    attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
    attr[1].val.accessPolicyWindow.base_ptr = ring;
    attr[1].val.accessPolicyWindow.num_bytes = rb;
    attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
    attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cfg.numAttrs = 2;
    return cudaLaunchKernelExC(&cfg, (const void*)k, args);
}

template <bool INV, int NS, int MINB>
cudaError_t ab8_t(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw, void* ws,
                  size_t ws_bytes, cudaStream_t st) {
    constexpr size_t SMEM = AbWs8Cfg<NS>::SMEM;
    auto k = k_ab_ws8<INV, NS, MINB>;
    AbGeom g;
    cudaError_t e = ab8_geom<INV, NS, MINB>(&g);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    if (!ws || ws_bytes < ab_ws_bytes(g.ring, batch)) return cudaErrorInvalidValue;
    void* ring = ws;
    int* ctl = reinterpret_cast<int*>((char*)ws + (size_t)g.ring * 65536 * sizeof(float2));
    CUtensorMap m_x, m_out, m_yst, m_yld;
    if (!encode3(&m_x, const_cast<void*>(in), 256, 256, (uint64_t)batch, 8, 256, 0) ||
        !encode3(&m_out, out, 256, 256, (uint64_t)batch, 8, 256, 64) ||
        !encode3(&m_yst, ring, 256, 256, g.ring, 8, 256, 0) || !encode3(&m_yld, ring, 256, 256, g.ring, 256, 8, 0))
        return cudaErrorInvalidValue;
    e = cudaMemsetAsync(ctl, 0, sizeof(int) * 2 * batch, st);
    if (e != cudaSuccess) return e;
    AbBulkCtl c{ctl, ctl + batch, g.D, g.ring};
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256, 3);
    int64_t a_batch = batch;
    const float2* a_ring = reinterpret_cast<const float2*>(ring);
    static const int opts = [] {
        const char* v = getenv("B200FFT_AB_OPTS");
        return v ? atoi(v) : 16;  // 16 x d: L2 prefetch of the A tile d tasks ahead
    }();
    int a_opts = opts;
    void* args[] = {&m_x, &m_yst, &m_yld, &m_out, &a_batch, &a_scale, &a_tw4, &a_tw, &c, &a_ring, &a_opts};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)ab_launch_grid(g.grid, batch, g.D, 32, NS), 1, 1);
    cfg.blockDim = dim3(288, 1, 1);
    cfg.dynamicSmemBytes = SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static const bool persist = [] {
        const char* v = getenv("B200FFT_AB_PERSIST");
        return !(v && v[0] == '0');
    }();
    if (persist) {
        static bool limit_set = false;
        const size_t rb = (size_t)g.ring * 65536 * sizeof(float2);
        if (!limit_set) {
            int dev = 0, mx = 0;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
            cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, rb < (size_t)mx ? rb : (size_t)mx);
            limit_set = true;
        }
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = ring;
        attr[1].val.accessPolicyWindow.num_bytes = rb;
        attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelExC(&cfg, (const void*)k, args);
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
                          const void* tw, cudaStream_t st, void* ws, size_t ws_bytes) {
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
        case 16: return cluster2_t<float, 256, 256, 16, 16, 4, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        case 17: return cluster2_t<float, 256, 256, 16, 16, 3, INV, false, true>(in, out, batch, scale, tw4, tw, st);
        case 12: return cluster3_t<float, 3, INV>(in, out, batch, scale, tw4, tw, st);
        case 13: return step_ab_t<float, 16, 16, 16, 4, INV>(in, out, batch, scale, tw4, tw, st);
        case 14: return step_ab_t<float, 32, 32, 16, 2, INV>(in, out, batch, scale, tw4, tw, st);
        case 15: return fused_ab_t<float, INV>(in, out, batch, scale, tw4, tw, st);
        case 18: return cluster4_t<float, 2, INV>(in, out, batch, scale, tw4, tw, st);
        case 19: return cluster5_t<float, 4, INV>(in, out, batch, scale, tw4, tw, st);
        case 20: return cluster6_t<float, 4, INV, true>(in, out, batch, scale, tw4, tw, st);
        case 21: return cluster6_t<float, 4, INV, false>(in, out, batch, scale, tw4, tw, st);
        case 27: return cluster6_t<float, 5, INV, false>(in, out, batch, scale, tw4, tw, st);
        case 28: return ab_pipe_t<float, 3, INV>(in, out, batch, scale, tw4, tw, st);
        case 31: return cluster2_t<float, 256, 256, 16, 16, 6, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        case 40: return ab_bulk_t<INV>(in, out, batch, scale, tw4, tw, st);
        case 41: return ab_tma_t<INV>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 42: return ab_tma_t<INV, true>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 43: return ab_tma_t<INV, true, 6>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 44: return ab_tma_t<INV, true, 2>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 45: return ab8_t<INV, 4, 3>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 46: return ab8_t<INV, 3, 4>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 47: return ab_ds_t<INV>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
        case 29: return ab_pipe_t<float, 2, INV>(in, out, batch, scale, tw4, tw, st);
        case 30: return ab_pipe_t<float, 4, INV>(in, out, batch, scale, tw4, tw, st);
        case 22: return step_ab2_t<float, INV>(in, out, batch, scale, tw4, tw, st);
        case 23: return cluster2_t<float, 256, 256, 16, 16, 5, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        case 24: return cluster2_t<float, 256, 256, 16, 16, 3, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        case 25: return cluster2_t<float, 256, 256, 8, 16, 2, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        case 26: return cluster2_t<float, 256, 256, 8, 16, 3, INV, true, true>(in, out, batch, scale, tw4, tw, st);
        default: return cudaErrorInvalidValue;
    }
}

size_t cluster_workspace_bytes(int prec, int64_t n, int variant, int64_t batch) {
    if (prec != 0 || n != 65536 || variant < 41 || variant > 47) return 0;
    AbGeom g;
    cudaError_t e = variant == 47   ? ds_geom<false>(&g)
                    : variant == 45 ? ab8_geom<false, 4, 3>(&g)
                    : variant == 46 ? ab8_geom<false, 3, 4>(&g)
                    : variant == 42 ? ab_geom<false, true>(&g)
                    : variant == 43 ? ab_geom<false, true, 6>(&g)
                    : variant == 44 ? ab_geom<false, true, 2>(&g)
                                    : ab_geom<false, false>(&g);
    if (e != cudaSuccess) return 0;
    return ab_ws_bytes(g.ring, batch);
}

cudaError_t launch_cluster(int prec, bool inv, int64_t n, const void* in, void* out, int64_t batch,
                           double scale, const void* tw4, const void* tw, int variant, cudaStream_t st, void* ws,
                           size_t ws_bytes) {
    if (prec == 0 && n == 65536)
        return inv ? cluster_65536<true>(variant, in, out, batch, scale, tw4, tw, st, ws, ws_bytes)
                   : cluster_65536<false>(variant, in, out, batch, scale, tw4, tw, st, ws, ws_bytes);
    return cudaErrorInvalidValue;
}

}  // namespace b200fft
