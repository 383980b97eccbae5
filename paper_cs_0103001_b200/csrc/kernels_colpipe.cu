// kernels_colpipe.cu -- launcher of the one-pass column filter of the 8192-row
// Gaussian pipeline (fft_colpipe.cuh, C4 = BASELINE configs[3]).
#include <cudaTypedefs.h>

#include <cstdlib>

#include "fft_colpipe.cuh"
#include "launch.h"

namespace b200fft {

namespace {

bool encode3d(CUtensorMap* map, void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t s1, uint64_t s2,
              uint32_t b0, uint32_t b1, uint32_t b2) {
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

}  // namespace

bool colfilt_supported(int64_t N, int64_t M) {
    const char* v = getenv("B200FFT_PIPE_COLS1");
    if (v && v[0] == '0') return false;
    return N == 8192 && M >= 16 && (M & (M - 1)) == 0;
}

size_t colfilt_workspace_bytes(int64_t M, int64_t nimg) {
    return (size_t)2 * (M / 16) * nimg * sizeof(int) + 16;
}

cudaError_t launch_colfilt(void* grid, int64_t M, int64_t nimg, double scale, const void* tw, const void* tl,
                           const void* gu, const void* gv, int64_t col_off, void* ws, size_t ws_bytes,
                           cudaStream_t st) {
    constexpr int64_t N = 8192;
    if (nimg <= 0) return cudaSuccess;
    if (M < 16 || M % 16 || (M / 16) * nimg >= ((int64_t)1 << 30)) return cudaErrorInvalidValue;
    if (!ws || ws_bytes < colfilt_workspace_bytes(M, nimg)) return cudaErrorInvalidValue;
    int grid_n = 0;
    // tuning: B200FFT_COLFILT_TW = 1 (default): the A / A' step twiddles from
    // the constant table, 0: by recurrence (C4 0.8955 / 0.8997 ms; with the B
    // steps' from the table too, 1.043 ms: the B task then spills 300 B)
    const char* twv = getenv("B200FFT_COLFILT_TW");
    const int twm = twv ? atoi(twv) & 1 : 1;
    int cg_sh = 0;
    while (((int64_t)1 << cg_sh) < M / 16) ++cg_sh;
    const bool p2 = ((int64_t)1 << cg_sh) == M / 16;
    const void* kern = p2 ? (twm ? (const void*)k_colfilt<128, 1, true> : (const void*)k_colfilt<128, 0, true>)
                          : (twm ? (const void*)k_colfilt<128, 1, false> : (const void*)k_colfilt<128, 0, false>);
    cudaError_t e = kernel_setup(kern, 320, ColPipeCfg::SMEM, &grid_n);
    if (e == cudaSuccess) e = w256_upload();  // the constant step twiddles (fft_engine.cuh)
    if (e != cudaSuccess) return e;
    const int64_t groups = (M / 16) * nimg;
    int* ctr = reinterpret_cast<int*>(ws);
    unsigned long long* next =
        reinterpret_cast<unsigned long long*>((char*)ws + ((sizeof(int) * 2 * groups + 7) & ~(size_t)7));
    e = cudaMemsetAsync(ws, 0, ((sizeof(int) * 2 * groups + 7) & ~(size_t)7) + 8, st);
    if (e != cudaSuccess) return e;
    CUtensorMap ma, mb;
    // A / A': (col, n2, n1 + 64 img) -> ((64 img + n1) 128 + n2) M + col; box 16 x 4 x 64
    // B: (col, row) -> row M + col; box 16 x 256
    if (!encode3d(&ma, grid, (uint64_t)M, 128, (uint64_t)(64 * nimg), (uint64_t)M, (uint64_t)(128 * M), 16, 4, 64) ||
        !encode3d(&mb, grid, (uint64_t)M, (uint64_t)(N * nimg), 1, (uint64_t)M, (uint64_t)(N * nimg * M), 16, 256, 1))
        return cudaErrorInvalidValue;
    // phase distance: B(g) is 96 D positions after A(g), beyond the ~900
    // positions in flight; 2 D + ~10 groups (1 MiB each) live in L2
    const char* dv = getenv("B200FFT_COLS1_D");
    // (D = 24: C4 0.8095-0.8102 vs 0.8155-0.8167 ms at D = 32, same box,
    // alternating; 16: 0.830, 40: 0.868)
    ColPipeCtl c{ctr, ctr + groups, next, dv ? atoi(dv) : 24};
    float2* a_grid = reinterpret_cast<float2*>(grid);
    int64_t a_M = M, a_nimg = nimg;
    float a_scale = (float)scale;
    const float2* a_tw64 = reinterpret_cast<const float2*>(tw) + tw_base(64);
    const float2* a_tw128 = reinterpret_cast<const float2*>(tw) + tw_base(128);
    const float2* a_tl = reinterpret_cast<const float2*>(tl);
    const float* a_gu = reinterpret_cast<const float*>(gu);
    const float* a_gv = reinterpret_cast<const float*>(gv);
    int64_t a_off = col_off;
    // column groups per image: a power of two (mask / shift indexing, p2) or
    // not (32-bit division)
    void* args[] = {&ma, &mb, &a_grid, &a_M, &a_nimg, &a_scale, &a_tw64, &a_tw128, &a_tl, &a_gu, &a_gv, &a_off,
                    &cg_sh, &c};
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    const int64_t npos = (groups + 2 * (int64_t)c.D) * 96;
    cfg.gridDim = dim3((unsigned)(npos < grid_n ? npos : grid_n), 1, 1);
    cfg.blockDim = dim3(320, 1, 1);
    cfg.dynamicSmemBytes = ColPipeCfg::SMEM;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, kern, args);
}

// this module's copy of the constant step-twiddle table (fft_engine.cuh
// c_w256), uploaded at plan creation so no launch does it (graph capture)
cudaError_t colfilt_upload_constants() { return w256_upload(); }

}  // namespace b200fft
