// kernels_big.cu -- launcher of the two-pass 2^30-point transform
// (fft_big.cuh, C5 = BASELINE configs[4] on one GPU).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "fft_big.cuh"
#include "launch.h"

namespace b200fft {

namespace {

bool enc3(CUtensorMap* map, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2, uint32_t b0,
          uint32_t b1, uint32_t b2) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = [] {
        PFN_cuTensorMapEncodeTiled_v12000 f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return f;
    }();
    if (!enc) return false;
    const cuuint64_t dims[3] = {d0, d1, d2};
    const cuuint64_t strides[2] = {s1 * 8, s2 * 8};
    const cuuint32_t box[3] = {b0, b1, b2};
    const cuuint32_t es[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int big_d() {
    const char* v = getenv("B200FFT_BIG_D");
    return v ? atoi(v) : 6;
}
int big_ring() {
    const char* v = getenv("B200FFT_BIG_RING");
    return big_d() + (v ? atoi(v) : 6);
}

template <bool INV, int PASS>
cudaError_t big_pass(const void* in, void* out, double scale, const void* tw, const void* twl, const void* whi,
                     const void* wlo, void* ws, size_t ws_bytes, cudaStream_t st) {
    constexpr int64_t L = BigCfg::L, GROUPS = 2048;
    const int D = big_d(), R = big_ring();
    if (!ws || ws_bytes < big_workspace_bytes()) return cudaErrorInvalidValue;
    int grid_n = 0;
    const void* kern = (const void*)k_big<INV, PASS>;
    cudaError_t e = kernel_setup(kern, 320, BigCfg::SMEM, &grid_n);
    if (e == cudaSuccess) e = w256_upload();  // the constant step twiddles (fft_engine.cuh)
    if (e != cudaSuccess) return e;
    float2* ring = reinterpret_cast<float2*>(ws);
    int* ctr = reinterpret_cast<int*>((char*)ws + (size_t)R * BigCfg::SLOT * sizeof(float2));
    unsigned long long* next = reinterpret_cast<unsigned long long*>(ctr + 2 * GROUPS);
    e = cudaMemsetAsync(ctr, 0, sizeof(int) * 2 * GROUPS + 8, st);
    if (e != cudaSuccess) return e;
    CUtensorMap mi, mr;
    bool ok;
    if (PASS == 1) {
        // x [n2][n1]: (n1, a, c) -> (a + 128 c) N1 + n1; box 16 x 1 x 256
        ok = enc3(&mi, const_cast<void*>(in), (uint64_t)L, 128, 256, (uint64_t)L, (uint64_t)(128 * L), 16, 1, 256) &&
             // ring [kc][a][16]: (t, a, kc) ; box 16 x 128 x 2
             enc3(&mr, ring, 16, 128, (uint64_t)256 * R, 16, 2048, 16, 128, 2);
    } else {
        // Y rows: (a, c, row) -> row L + a + 128 c; box 16 x 256 x 1
        ok = enc3(&mi, const_cast<void*>(in), 128, 256, (uint64_t)L, 128, (uint64_t)L, 16, 256, 1) &&
             // ring [kc][r][128 a]: (a, r, kc) ; box 128 x 16 x 2
             enc3(&mr, ring, 128, 16, (uint64_t)256 * R, 128, 2048, 128, 16, 2);
    }
    if (!ok) return cudaErrorInvalidValue;
    BigCtl c{ctr, ctr + GROUPS, next, D, R};
    float a_scale = (float)scale;
    float2* a_ring = ring;
    float2* a_out = reinterpret_cast<float2*>(out);
    const float2* a_tw256 = reinterpret_cast<const float2*>(tw) + tw_base(256);
    const float2* a_tw128 = reinterpret_cast<const float2*>(tw) + tw_base(128);
    const float2* a_twl = reinterpret_cast<const float2*>(twl);
    const float2* a_hi = reinterpret_cast<const float2*>(whi);
    const float2* a_lo = reinterpret_cast<const float2*>(wlo);
    // B200FFT_BIG_XO (tuning): pass 1's Y stores 0 = evict-last, 1 = evict-first,
    // 2 = without a cache hint (default: C5 19.97 / 19.69 / 19.69 ms fwd + inv);
    // + 8: pass 2's X stores without a hint (else evict-first); + 4 / + 16:
    // timing experiments, pass 2's X / pass 1's Y stored as contiguous blocks
    // (wrong order)
    static const int xo = [] {
        const char* v = getenv("B200FFT_BIG_XO");
        return v ? atoi(v) : 2;
    }();
    int a_xo = xo;
    void* args[] = {&mi, &mr, &a_ring, &a_out, &a_scale, &a_tw256, &a_tw128, &a_twl, &a_hi, &a_lo, &c, &a_xo};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.gridDim = dim3((unsigned)grid_n, 1, 1);
    cfg.blockDim = dim3(320, 1, 1);
    cfg.dynamicSmemBytes = BigCfg::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // the ring persisting in L2 (set-aside = ring): consumed rows are
    // overwritten in L2 by the slot's next group instead of being written back
    // (without it: +4.3 GB of DRAM writes per pass, ncu)
    const char* pv = getenv("B200FFT_BIG_PERSIST");
    if (!(pv && pv[0] == '0')) {
        int dev = 0;
        cudaGetDevice(&dev);
        const size_t rb = (size_t)R * BigCfg::SLOT * sizeof(float2);
        l2_persist_request(dev, rb);
        attr[1].id = cudaLaunchAttributeAccessPolicyWindow;
        attr[1].val.accessPolicyWindow.base_ptr = ring;
        attr[1].val.accessPolicyWindow.num_bytes = rb;
        attr[1].val.accessPolicyWindow.hitRatio = 1.0f;
        attr[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        attr[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cfg.numAttrs = 2;
    }
    return cudaLaunchKernelExC(&cfg, kern, args);
}

}  // namespace

bool big_supported(int prec, int64_t n) {
    const char* v = getenv("B200FFT_C5_2PASS");
    if (v && v[0] == '0') return false;
    return prec == 0 && n == ((int64_t)1 << 30);
}

size_t big_workspace_bytes() {
    return (size_t)big_ring() * BigCfg::SLOT * sizeof(float2) + sizeof(int) * 2 * 2048 + 16;
}

cudaError_t launch_big(bool inv, const void* in, void* mid, void* out, double scale, const void* tw, const void* twl,
                       const void* whi, const void* wlo, void* ws, size_t ws_bytes, cudaStream_t st) {
    cudaError_t e = inv ? big_pass<true, 1>(in, mid, 1.0, tw, twl, whi, wlo, ws, ws_bytes, st)
                        : big_pass<false, 1>(in, mid, 1.0, tw, twl, whi, wlo, ws, ws_bytes, st);
    if (e != cudaSuccess) return e;
    return inv ? big_pass<true, 2>(mid, out, scale, tw, twl, whi, wlo, ws, ws_bytes, st)
               : big_pass<false, 2>(mid, out, scale, tw, twl, whi, wlo, ws, ws_bytes, st);
}

// this module's copy of the constant step-twiddle table (fft_engine.cuh
// c_w256), uploaded at plan creation so no launch does it (graph capture)
cudaError_t big_upload_constants() { return w256_upload(); }

}  // namespace b200fft
