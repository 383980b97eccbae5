// launch.h -- internal launchers of libb200fft (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace b200fft {

struct FilterArgs;

// Base pointers of the column blocks of a blocked row layout (the all-to-all
// layout of the slab-decomposed 2D transform): element (row, v) of a launch
// with shift sh lives at ((C*)p[v >> sh])[(row << sh) | (v & (2^sh - 1))].
// The blocks may be local slabs or PEER memory (CUDA IPC over NVLink): the
// row pass then stores its blocks straight into the other ranks' receive
// slabs and the final row pass loads them from there -- the all-to-alls are
// fused into the row kernels (Multi-GPU).
constexpr int kMaxBlocks = 16;
struct BlockPtrs {
    void* p[kMaxBlocks];
};

// Programmatic dependent launch of the per-CTA kernels (B200FFT_PDL=0: off);
// every such kernel starts with B200FFT_PDL_PROLOGUE (fft_common.cuh).  It
// is applied only where it measured faster (PdlScope around those launches:
// the image application's chain of short kernels; the C4 chain of column
// passes measured 12% slower with it).
bool pdl_enabled();
bool& pdl_hint();  // thread-local: launches inside a PdlScope use PDL
struct PdlScope {
    bool saved;
    PdlScope() : saved(pdl_hint()) { pdl_hint() = true; }
    ~PdlScope() { pdl_hint() = saved; }
};
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    if (!pdl_enabled() || !pdl_hint()) {
        kern<<<grid, block, smem, st>>>(args...);
        return cudaGetLastError();
    }
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Largest transform length handled by one CTA, per precision (0 = c64, 1 = c128).
constexpr int64_t kRowsMax = 8192;
constexpr int64_t kColsMax[2] = {8192, 4096};

// Kernel family A: batch contiguous rows of length R (power of two <= 8192).
// in_sh / out_sh >= 0: rows stored in column blocks of 2^sh (all-to-all pack
// layout): block q at in_blocks->p[q] / out_blocks->p[q], or, when null, at
// in / out + q * (batch << sh) elements; -1: natural row-major.
// rowfilt (T[R], optional): the separable-pipeline row pass, forward ->
// * rowfilt[v] * scale -> inverse, stored unscaled (inv must be false).
cudaError_t launch_rows(int prec, bool inv, bool real_in, int64_t R, const void* in, void* out,
                        int64_t batch, double scale, const void* tw, cudaStream_t st, int in_sh = -1,
                        int out_sh = -1, const void* rowfilt = nullptr, const BlockPtrs* in_blocks = nullptr,
                        const BlockPtrs* out_blocks = nullptr);

// Separable-pipeline pass with a transposed store (complex64, 256 <= R <=
// 2048): rows of length R -> forward -> * rowfilt[v] * scale -> inverse ->
// out[v][row] (leading dimension batch).  Two of these (rows, then the rows
// of the transposed grid) are the whole Gaussian pipeline.
bool rows_filter_transposed_supported(int prec, int64_t R);
// pair = 1 (NEXT-3): `in` holds 2 batch real float32 rows, transformed
// two at a time as one complex row (a + i b); out is the transposed real
// grid [R][2 batch] (the row filter must be real and even).  pair = 2: the
// same, out is the transposed complex grid with zero imaginary parts.
// pdl: programmatic dependent launch (the second pass of a pipeline starts
// on the SMs the first one leaves and waits for its results on the device).
cudaError_t launch_rows_filter_transposed(bool real_in, int64_t R, const void* in, void* out, int64_t batch,
                                          double scale, const void* tw, const void* rowfilt, cudaStream_t st,
                                          int pair = 0, bool pdl = false);

// Both passes of the real-pair pipeline of a square R x R grid (512 <= R
// <= 2048, complex64) in one cooperative launch (k_rows_tma2): in (R real
// rows) -> pass 1 (row pairs, fwd * filt1 * scale1 * inv) -> mid (the
// transposed real grid, R x R floats) -> grid barrier -> pass 2 (filt2,
// scale2) -> out (pair2 = 2: the complex grid, imaginary parts 0; the only
// form built).
// gbar: a device counter that only grows (zeroed once); *gen: the host's
// launch count for it (incremented here).
bool rows_filter2_supported(int prec, int64_t N, int64_t M);
cudaError_t launch_rows_filter2(int64_t R, const void* in, void* mid, void* out, double scale1, const void* filt1,
                                double scale2, const void* filt2, const void* tw, int pair2, unsigned long long* gbar,
                                cudaStream_t st);

// Kernel family B: column transforms of nimg grids [R][S]; mode 0 fwd, 1 inv,
// 2 fwd -> filter*scale -> inv.
cudaError_t launch_cols(int prec, int mode, int64_t R, const void* in, void* out, int64_t S,
                        int64_t nimg, double scale, const void* tw, const FilterArgs& f,
                        cudaStream_t st);

// The column direction of the 2D pipeline as a four-step (complex64,
// 64 <= R <= 4096, k_cols_pipe): mode 3 = forward DFT over R rows + twiddle
// W_L^{(col / f.tdiv) u}, mode 4 = conj twiddle + inverse DFT, mode 2 with
// f.kind 6 = fwd * g[img + f.n1 u] * scale * inv.
cudaError_t launch_cols_fourstep(int mode, int64_t R, const void* in, void* out, int64_t S, int64_t nimg,
                                 double scale, const void* tw, const FilterArgs& f, cudaStream_t st);

// Kernel family C: one global Stockham pass of radix R (128..1024) over
// `batch` rows of length L with span Ns; pa/pb: the pass twiddle tables
// (pa[r][k mod 2^klo_sh], pb[r][k >> klo_sh]).
cudaError_t launch_pass(int prec, bool inv, int64_t R, const void* in, void* out, int64_t L,
                        int64_t Ns, int64_t batch, double scale, const void* tw, const void* pa,
                        const void* pb, int klo_sh, cudaStream_t st);

// Distributed four-step helpers (kernels_misc.cu): batched transpose
// out[c][r] = in[r][c] of nmat [R][Cn] matrices; four-step twiddle
// y[row][k2] *= W_N^{(row0 + row) k2} with W_N^x = ta[x >> sh] * tb[x & mask].
// Distributed transpose G[P R][Cn] (row slabs of R at src.p[s]) -> G^T
// (row slabs of Cb at dst.p[d]) over global rows [row0, +nrows) x columns
// [col0, +ncols) (kernels_misc.cu k_dist_transpose).
cudaError_t launch_dist_transpose(int prec, const BlockPtrs& src, const BlockPtrs& dst, int64_t R, int64_t Cn,
                                  int64_t Cb, int64_t P, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
                                  cudaStream_t st);
cudaError_t launch_transpose(int prec, const void* in, void* out, int64_t R, int64_t Cn, int64_t nmat,
                             cudaStream_t st);
cudaError_t launch_twiddle4(int prec, bool inv, void* y, int64_t rows, int64_t L, int64_t row0, const void* ta,
                            const void* tb, int sh, cudaStream_t st);

// The paper's image application (kernels_image.cu): row DFTs of the N x M
// grid of `nrows` = batch * N rows of length M.  Forward: u8 [batch][h][w]
// zero-padded to [N][M] in the load -> complex64 out.  Inverse: complex64 in
// -> real part, round half up, clamp [0, max_val], crop to h x w -> u8 out.
cudaError_t launch_image_rows(bool inv, int64_t M, const void* in, void* out, int64_t nrows, int64_t N, int64_t h,
                              int64_t w, int max_val, const void* tw, cudaStream_t st);

// The paper's tree combine (NEXT-2, kernels_misc.cu k_tree_combine): nb
// radix-2 combines of E, O (length M, stride es) into Y (length 2M, stride
// ys) with W_{2M}^k = ta[x >> sh] * tb[x & mask], x = k * xstep.
cudaError_t launch_tree_combine(int prec, const void* e, const void* o, void* y, int64_t M, int64_t nb, int64_t es,
                                int64_t ys, int64_t xstep, const void* ta, const void* tb, int sh, cudaStream_t st);

// Real-input / real-output rows (kernels_real.cu, fft_real.cuh, NEXT-3):
// batch rows of M reals (float for prec 0, double for 1) <-> rows of M/2 + 1
// complex bins (Hermitian half spectrum), out = scale * (forward sum e^-,
// or for C2R the unscaled inverse sum e^+).  rtw: W_M^k, k < M/2.  2 <= M <= 8192.
// ld: row stride of the half spectrum in bins (<= 0: M/2 + 1, the API layout;
// the internal pipeline pads it to a multiple of 16 for k_colfilt).
cudaError_t launch_rows_r2c(int prec, int64_t M, const void* in, void* out, int64_t batch, double scale,
                            const void* tw, const void* rtw, cudaStream_t st, int64_t ld = -1);
cudaError_t launch_rows_c2r(int prec, int64_t M, const void* in, void* out, int64_t batch, double scale,
                            const void* tw, const void* rtw, cudaStream_t st, int64_t ld = -1);

// One-pass column filter of the 8192-row Gaussian pipeline (kernels_colpipe.cu,
// fft_colpipe.cuh): in place on [nimg][8192][M] complex64 (M % 16 == 0),
// column operator IDFT_N(g_N(u) * scale * [g_M(v + col_off)] * DFT_N); tl =
// W_N^x (x < N), gu = g_N (N floats), gv = g_M or null; ws: counters.
// colfilt_supported: the pipelines' power-of-two widths; any M % 16 == 0
// (e.g. a padded half spectrum) is accepted by launch_colfilt.
bool colfilt_supported(int64_t N, int64_t M);
size_t colfilt_workspace_bytes(int64_t M, int64_t nimg);
cudaError_t launch_colfilt(void* grid, int64_t M, int64_t nimg, double scale, const void* tw, const void* tl,
                           const void* gu, const void* gv, int64_t col_off, void* ws, size_t ws_bytes,
                           cudaStream_t st);

// Two-pass 2^30-point complex64 transform (kernels_big.cu, fft_big.cuh, C5 on
// one GPU): in -> mid (pass 1: column FFTs + four-step twiddle) -> out (pass 2:
// row FFTs, x scale); mid must not alias in or out; twl = W_32768^x, whi /
// wlo = W_n^{i 32768} / W_n^i (i < 32768); ws: the L2 ring and counters.
bool big_supported(int prec, int64_t n);
size_t big_workspace_bytes();
cudaError_t launch_big(bool inv, const void* in, void* mid, void* out, double scale, const void* tw, const void* twl,
                       const void* whi, const void* wlo, void* ws, size_t ws_bytes, cudaStream_t st);

// Per-device, thread-safe one-time kernel setup: sets `kern`'s dynamic
// shared-memory limit on the current device (once per device) and, if
// grid_max != nullptr, returns its persistent grid there (SM count x
// occupancy at `threads` threads and `smem` bytes).  (kernels_misc.cu)
cudaError_t kernel_setup(const void* kern, int threads, size_t smem, int* grid_max);

// One-pass 65536- and 32768-point complex64 transforms (fft_c2.cuh, C2):
// n = N1 * 256 (N1 = 256, 128) four-step through an L2-resident ring.  tw4:
// W_n^{n1 k2} laid out [k2][n1]; caller-provided scratch of
// c2_workspace_bytes (the ring and the task counters).
bool c2_supported(int prec, int64_t n, int* n1, int* n2);
size_t c2_workspace_bytes(int64_t batch, int64_t n);
// plan lifetime bookkeeping: the device's persisting-L2 set-aside for the
// ring is released with its last 65536-point plan
void c2_plan_acquire(int dev);
void c2_plan_release(int dev);
// the device's persisting-L2 set-aside for an L2 ring of ring_bytes (the
// largest requested; released with the last acquiring plan)
void l2_persist_request(int dev, size_t ring_bytes);
// ow_a / ow_b / ow_sh / ow_row0: optional outer four-step twiddle W_n^{(row0
// + b) k} on output k of transform b (n = 32768 only; ow_a = nullptr: none)
cudaError_t launch_c2(bool inv, int64_t n, const void* in, void* out, int64_t batch, double scale, const void* tw4,
                      const void* tw, void* ws, size_t ws_bytes, cudaStream_t st, const void* ow_a = nullptr,
                      const void* ow_b = nullptr, int ow_sh = 0, int64_t ow_row0 = 0);

// the constant step-twiddle tables of the task-pipeline modules (one copy per
// module, fft_engine.cuh c_w256), uploaded for the current device
cudaError_t c2_upload_constants();
cudaError_t big_upload_constants();
cudaError_t colfilt_upload_constants();

}  // namespace b200fft
