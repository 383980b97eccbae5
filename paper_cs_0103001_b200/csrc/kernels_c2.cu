// kernels_c2.cu -- launcher of the one-pass 65536-point transform
// (fft_c2.cuh, C2 = BASELINE configs[1]).
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "fft_c2.cuh"
#include "fft_c2pair.cuh"
#include "launch.h"

namespace b200fft {

namespace {

// tensor maps (cuTensorMapEncodeTiled through the runtime's driver entry
// point: no libcuda link); 3D views [d2][d1][d0] of 8-byte elements
bool encode3(CUtensorMap* map, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0, uint32_t b1,
             int swz) {  // swz: 0 or 128 (the B output box's TMA swizzle span)
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return f;
    }();  // thread-safe one-time initialisation (C++11 magic static)
    if (!enc) return false;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {d0 * 8, d0 * d1 * 8};
    const cuuint32_t box[3] = {b0, b1, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// launch geometry per (device, direction): persistent grid, dependency
// distance D (transforms) and ring slots; also whether the device's
// persisting-L2 set-aside has been sized for the ring.  Guarded by a mutex:
// plans on different threads / devices may launch concurrently.
// The kernel: k_ab_st (default: direct stores from registers, 2 stages,
// 3 CTAs/SM, dynamic task order) or k_ab_ws (the round-1 kernel: TMA stores
// from the stage, static order), B200FFT_C2 = "st" | "ws" (read at each
// launch, so the tests cover both).
enum C2Kind { C2_WS = 0, C2_ST = 1, C2_NKIND = 2 };
int c2_kind() {
    const char* v = getenv("B200FFT_C2");
    if (v && !strcmp(v, "ws")) return (int)C2_WS;
    return (int)C2_ST;
}
const void* c2_kernel(int kind, bool inv, int64_t n = 65536, bool otw = false) {
    if (n == 32768 && otw)
        return inv ? (const void*)k_ab_st<true, 2, 3, 32768, true> : (const void*)k_ab_st<false, 2, 3, 32768, true>;
    if (n == 32768) return inv ? (const void*)k_ab_st<true, 2, 3, 32768> : (const void*)k_ab_st<false, 2, 3, 32768>;
    if (kind == C2_ST) return inv ? (const void*)k_ab_st<true, 2, 3> : (const void*)k_ab_st<false, 2, 3>;
    return inv ? (const void*)k_ab_ws<true> : (const void*)k_ab_ws<false>;
}
int c2_threads(int kind) { return kind == C2_WS ? 288 : 320; }
size_t c2_smem(int kind) { return kind == C2_WS ? AbWsCfg::SMEM : AbStCfg<2>::SMEM; }

// launch geometry per device: persistent grid per (kernel, direction), and
// the dependency distance D (transforms) and ring slots shared by all of them
// (one workspace size); also whether the device's persisting-L2 set-aside
// has been sized for the ring.  Guarded by a mutex: plans on different
// threads / devices may launch concurrently.
struct AbGeom {
    int grid[C2_NKIND][2] = {};  // [kind][inverse]
    int grid32[2][2] = {};       // k_ab_st<32768>: [outer twiddle][inverse]
    int D = 0, ring = 0;
    bool limit_set = false;
    size_t limit = 0;  // the persisting set-aside requested so far (the largest ring)
    int plans = 0;     // live plans with an L2 ring on the device (c2_plan_acquire / release)
};
std::mutex g_geom_mu;
std::map<int, AbGeom> g_geom;

cudaError_t ab_geom(int dev, AbGeom* g) {
    std::lock_guard<std::mutex> lk(g_geom_mu);
    AbGeom& c = g_geom[dev];
    if (!c.ring) {
        AbGeom t;
        int sms = 0, gmax = 0;
        cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        for (int kind = 0; kind < C2_NKIND && e == cudaSuccess; ++kind)
            for (int d = 0; d < 2 && e == cudaSuccess; ++d) {
                const void* k = c2_kernel(kind, d != 0);
                int occ = 0;
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2_smem(kind));
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, c2_threads(kind), c2_smem(kind));
                t.grid[kind][d] = sms * (occ > 0 ? occ : 1);
                gmax = t.grid[kind][d] > gmax ? t.grid[kind][d] : gmax;
            }
        for (int o = 0; o < 2 && e == cudaSuccess; ++o)
            for (int d = 0; d < 2 && e == cudaSuccess; ++d) {
                const void* k = c2_kernel(C2_ST, d != 0, 32768, o != 0);
                int occ = 0;
                e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c2_smem(C2_ST));
                if (e == cudaSuccess)
                    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, c2_threads(C2_ST), c2_smem(C2_ST));
                t.grid32[o][d] = sms * (occ > 0 ? occ : 1);
            }
        if (e != cudaSuccess) return e;
        // every wait must point at least (tasks in flight per CTA) x grid
        // positions back in the task order: NS = 2 per CTA for k_ab_ws
        // (B200FFT_AB_D / B200FFT_AB_RING: tuning knobs for the margins)
        const char* dv = getenv("B200FFT_AB_D");
        const char* rv = getenv("B200FFT_AB_RING");
        t.D = (2 * gmax + 15) / 16 + (dv ? atoi(dv) : 8);
        // ring = D + 40 slots: an A load waits on the B parts 40 transforms
        // (1280 task positions) back, always an earlier task and beyond the
        // ~900 positions in flight (D + 8 / 24 / 40 / 56: 1.17 / 1.007 / 0.968
        // / 0.971 ms; rings above ~110 slots (55 MB) exceed the persisting L2
        // set-aside and spill: 1.26 ms)
        t.ring = t.D + (rv ? atoi(rv) : 40);
        if (getenv("B200FFT_VERBOSE"))
            fprintf(stderr, "c2: device %d grids ws %d st %d, D %d, ring %d, kernel %d\n", dev, t.grid[0][0],
                    t.grid[1][0], t.D, t.ring, c2_kind());
        c = t;
    }
    *g = c;
    return cudaSuccess;
}

// The persisting-L2 set-aside of a device, sized once for the ring
}  // namespace

// The device's persisting-L2 set-aside, sized for the largest ring asked for
// (the 65536-point ring, the 2^30 transform's ring); set on first use.
void l2_persist_request(int dev, size_t ring_bytes) {
    std::lock_guard<std::mutex> lk(g_geom_mu);
    AbGeom& c = g_geom[dev];
    if (c.limit_set && c.limit >= ring_bytes) return;
    int mx = 0;
    cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, dev);
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur == dev) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, ring_bytes < (size_t)mx ? ring_bytes : (size_t)mx);
    c.limit_set = true;
    c.limit = ring_bytes;
}

namespace {

void ab_persist_limit(int dev, size_t ring_bytes) { l2_persist_request(dev, ring_bytes); }

// caller-provided scratch: the Y ring (ring x L x 8 B), then the counters
size_t ab_ws_bytes(int64_t ring, int64_t batch, int64_t n = 65536) {
    return (size_t)ring * n * sizeof(float2) + (size_t)2 * batch * sizeof(int) + 16;
}
// the N = 32768 form has half the tasks per transform and half-size slots:
// twice the dependency distance and ring slots for the same positions / bytes
int64_t ab_scale(int64_t n) { return n == 32768 ? 2 : 1; }

// Grid of one launch.  A CTA's A task at local index k is signalled
// (done_a) only once its producer has issued its loads up to local index
// k + NS - 1 (or its last one), i.e. task position j + (NS - 1) grid.  A B
// load at position i waits for A parts at positions j <= i - d, so the
// schedule is deadlock-free when every such distance d exceeds (NS - 1)
// grid: in the steady state d >= 16 D + 1 (D is sized for it, ab_geom); with
// fewer transforms than D every A precedes every B and d >= 16 (batch - 1) +
// 1, so the grid is capped there -- unless every CTA holds at most one task.
int64_t ab_launch_grid(int64_t grid, int64_t batch, int64_t D, int NS) {
    const int64_t tasks = 32 * batch;
    if (tasks <= grid) return tasks;
    if (batch >= D || NS <= 1 || getenv("B200FFT_AB_NOCAP")) return grid;
    const int64_t cap = (16 * (batch - 1)) / (NS - 1);  // (NS - 1) g <= 16 (batch - 1) < d
    return cap < 1 ? 1 : (cap < grid ? cap : grid);
}

// k_ab_ws's tuning bits (B200FFT_AB_OPTS; default = the measured best, 144):
// bits 4..6 = L2 tensor prefetch of the A tile d tasks ahead (d = 1: -1.3%);
// bit 7 = A twiddles by a 15-step product from two table entries instead of
// 16 loads (-4.5%).  k_ab_st takes only experiment bits (B200FFT_AB_XOPTS,
// honoured only with B200FFT_ALLOW_WRONG=1; profiles/README.md "C2 bound"):
// wrong results: 1 = no loads / dependency waits, 2 = no stores, 4 = no
// dependency waits, 8 = no FFT arithmetic, 64 = no step-0 -> 1 exchange,
// 2048 = each B task stores one contiguous 32 KiB block; correct results:
// 16 = static round-robin positions, 32 = two positions per atomic, 128 /
// 256 / 1024 = X stores evict-first / .cs / evict-last (default: no hint),
// 512 = A loads evict-last, 4096 = step-1 twiddles by the recurrence (the
// earlier form, 3% slower) instead of the constant table, 16384 = Y stores
// with the evict-last hint (the earlier form, 1.3% slower).
int ab_opts(int kind) {
    if (kind == C2_WS) {
        const char* v = getenv("B200FFT_AB_OPTS");
        return v ? atoi(v) : (128 | 16);
    }
    const char* w = getenv("B200FFT_ALLOW_WRONG");
    const char* x = getenv("B200FFT_AB_XOPTS");
    return (w && w[0] == '1' && x) ? atoi(x) : 0;
}

template <bool INV, int64_t L = 65536>
cudaError_t ab_launch(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                      void* ws, size_t ws_bytes, cudaStream_t st, OuterTw ow = OuterTw{}) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    AbGeom g;
    e = ab_geom(dev, &g);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    constexpr int64_t N1 = L / 256;  // columns of the [256][N1] view (n = n1 + N1 n2)
    const int64_t D = g.D * ab_scale(L), R = g.ring * ab_scale(L);
    if (!ws || ws_bytes < ab_ws_bytes(R, batch, L)) return cudaErrorInvalidValue;
    if ((e = w256_upload()) != cudaSuccess) return e;
    void* ring = ws;
    const size_t rb = (size_t)R * L * sizeof(float2);
    int* ctl = reinterpret_cast<int*>((char*)ws + rb);
    const int kind = L == 65536 ? c2_kind() : (int)C2_ST;
    CUtensorMap m_x, m_out, m_yst, m_yld;
    if (!encode3(&m_x, const_cast<void*>(in), N1, 256, (uint64_t)batch, 16, 256, 0) ||
        !encode3(&m_out, out, 256, 256, (uint64_t)batch, 16, 256, 128) ||
        !encode3(&m_yst, ring, 256, 256, R, 16, 256, 0) ||
        !encode3(&m_yld, ring, N1, 256, R, (uint32_t)N1, (uint32_t)(4096 / N1), 0))
        return cudaErrorInvalidValue;
    // counters: done_a[batch], done_b[batch], then the 8-B task counter
    // (8-B aligned: 2 batch ints after the 512 KiB-aligned ring, padded)
    unsigned long long* next =
        reinterpret_cast<unsigned long long*>((char*)ctl + ((sizeof(int) * 2 * batch + 7) & ~(size_t)7));
    e = cudaMemsetAsync(ctl, 0, ((sizeof(int) * 2 * batch + 7) & ~(size_t)7) + 8, st);
    if (e != cudaSuccess) return e;
    AbCtl c{ctl, ctl + batch, next, (int)D, (int)R};
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256);
    int64_t a_batch = batch;
    int a_opts = ab_opts(kind);
    float2* a_ring = reinterpret_cast<float2*>(ring);
    float2* a_out = reinterpret_cast<float2*>(out);
    void* args_ws[] = {&m_x, &m_yst, &m_yld, &m_out, &a_batch, &a_scale, &a_tw4, &a_tw, &c, &a_opts};
    OuterTw a_ow = ow;
    void* args_st[] = {&m_x, &m_yld, &a_ring, &a_out, &a_batch, &a_scale, &a_tw4, &a_tw, &c, &a_opts, &a_ow};
    const int grid = L == 65536 ? g.grid[kind][INV ? 1 : 0] : g.grid32[ow.a != nullptr][INV ? 1 : 0];
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    // k_ab_st signals an A task as soon as its own stores are done (no
    // signal waits for a later load): no small-batch grid cap
    const int64_t tasks = 2 * (N1 / 16) * batch;
    cfg.gridDim = dim3((unsigned)(kind == C2_WS ? ab_launch_grid(grid, batch, g.D, AbWsCfg::NS)
                                                : (tasks < grid ? tasks : grid)),
                       1, 1);
    cfg.blockDim = dim3(c2_threads(kind), 1, 1);
    cfg.dynamicSmemBytes = c2_smem(kind);
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // An L2 access-policy window marks the Y ring persisting for this launch
    // (with a device persisting-L2 set-aside of the ring's size): the ring
    // then never spills to HBM (ncu: DRAM bytes = algorithmic + 1.3%, 1.10
    // -> 1.07 ms).  B200FFT_AB_PERSIST=0 turns it off.
    static const bool persist = [] {
        const char* v = getenv("B200FFT_AB_PERSIST");
        return !(v && v[0] == '0');
    }();
    if (persist) {
        ab_persist_limit(dev, rb);
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = ring;
        attr[1].val.accessPolicyWindow.num_bytes = rb;
        attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelExC(&cfg, c2_kernel(kind, INV, L, ow.a != nullptr), kind == C2_WS ? args_ws : args_st);
}

// k_ab_pair (fft_c2pair.cuh): one 2-CTA cluster per transform, Y in TMEM;
// grid = 2 x the co-resident clusters (at most one per transform)
std::mutex g_pair_mu;
std::map<int, int> g_pair_clusters;  // [device] -> co-resident 2-CTA clusters

template <bool INV>
cudaError_t pair_launch(const void* in, void* out, int64_t batch, double scale, const void* tw4, const void* tw,
                        cudaStream_t st) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (batch <= 0) return cudaSuccess;
    if ((e = w256_upload()) != cudaSuccess) return e;
    const void* kern = (const void*)k_ab_pair<INV>;
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(PairCfg::THREADS, 1, 1);
    cfg.dynamicSmemBytes = PairCfg::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int ncl = 0;
    {
        std::lock_guard<std::mutex> lk(g_pair_mu);
        auto it = g_pair_clusters.find(dev * 2 + (INV ? 1 : 0));
        if (it == g_pair_clusters.end()) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)PairCfg::SMEM);
            if (e != cudaSuccess) return e;
            cfg.gridDim = dim3(296, 1, 1);
            e = cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
            if (e != cudaSuccess) return e;
            if (ncl < 1) return cudaErrorInvalidConfiguration;
            g_pair_clusters[dev * 2 + (INV ? 1 : 0)] = ncl;
            if (getenv("B200FFT_VERBOSE")) fprintf(stderr, "c2 pair: device %d, %d clusters of 2\n", dev, ncl);
        } else {
            ncl = it->second;
        }
    }
    const int64_t npairs = batch < ncl ? batch : ncl;
    cfg.gridDim = dim3((unsigned)(2 * npairs), 1, 1);
    CUtensorMap m_x;
    if (!encode3(&m_x, const_cast<void*>(in), 256, 256, (uint64_t)batch, 16, 256, 0)) return cudaErrorInvalidValue;
    float a_scale = (float)scale;
    const float2* a_tw4 = reinterpret_cast<const float2*>(tw4);
    const float2* a_tw = reinterpret_cast<const float2*>(tw) + tw_base(256);
    int64_t a_batch = batch;
    float2* a_out = reinterpret_cast<float2*>(out);
    const char* w = getenv("B200FFT_ALLOW_WRONG");
    const char* x = getenv("B200FFT_PAIR_XO");
    int a_xo = (w && w[0] == '1' && x) ? atoi(x) : 0;
    void* args[] = {&m_x, &a_out, &a_batch, &a_scale, &a_tw4, &a_tw, &a_xo};
    return cudaLaunchKernelExC(&cfg, kern, args);
}

bool c2_pair_selected() {
    const char* v = getenv("B200FFT_C2");
    return v && !strcmp(v, "pair");
}

}  // namespace

bool c2_supported(int prec, int64_t n, int* n1, int* n2) {
    if (prec != 0 || (n != 65536 && n != 32768)) return false;
    const char* v = getenv("B200FFT_NO_AB32K");  // "1": 32768-point rows by the Stockham passes instead
    if (n == 32768 && v && v[0] == '1') return false;
    *n1 = (int)(n / 256);
    *n2 = 256;
    return true;
}

// The persisting-L2 set-aside and the ring's persisting lines are released
// when the device's last 65536-point plan is destroyed: they would otherwise
// keep ~50 MB of L2 from every later kernel (C4 / C5 measured 20% slower
// after a C2 run without this).
void c2_plan_acquire(int dev) {
    std::lock_guard<std::mutex> lk(g_geom_mu);
    ++g_geom[dev].plans;
}
void c2_plan_release(int dev) {
    std::lock_guard<std::mutex> lk(g_geom_mu);
    AbGeom& c = g_geom[dev];
    if (--c.plans > 0 || !c.limit_set) return;
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != dev) cudaSetDevice(dev);
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
    if (cur != dev && cur >= 0) cudaSetDevice(cur);
    c.limit_set = false;
    c.limit = 0;
}

size_t c2_workspace_bytes(int64_t batch, int64_t n) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    AbGeom g;
    if (ab_geom(dev, &g) != cudaSuccess) return 0;
    return ab_ws_bytes(g.ring * ab_scale(n), batch, n);
}

cudaError_t launch_c2(bool inv, int64_t n, const void* in, void* out, int64_t batch, double scale, const void* tw4,
                      const void* tw, void* ws, size_t ws_bytes, cudaStream_t st, const void* ow_a, const void* ow_b,
                      int ow_sh, int64_t ow_row0) {
    if (n == 32768) {
        const OuterTw ow{reinterpret_cast<const float2*>(ow_a), reinterpret_cast<const float2*>(ow_b), ow_sh,
                         ow_row0};
        return inv ? ab_launch<true, 32768>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st, ow)
                   : ab_launch<false, 32768>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st, ow);
    }
    if (ow_a) return cudaErrorInvalidValue;  // the outer twiddle is fused for 32768-point rows only
    if (c2_pair_selected())
        return inv ? pair_launch<true>(in, out, batch, scale, tw4, tw, st)
                   : pair_launch<false>(in, out, batch, scale, tw4, tw, st);
    return inv ? ab_launch<true>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st)
               : ab_launch<false>(in, out, batch, scale, tw4, tw, ws, ws_bytes, st);
}

// this module's copy of the constant step-twiddle table (fft_engine.cuh
// c_w256), uploaded at plan creation so no launch does it (graph capture)
cudaError_t c2_upload_constants() { return w256_upload(); }

}  // namespace b200fft
