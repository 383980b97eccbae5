// kernels_misc.cu -- the data-movement and twiddle kernels of the distributed
// four-step 1D transform (BASELINE configs[4]):
//   k_transpose : out[c][r] = in[r][c] for a batch of [R][Cn] matrices (the
//                 all-to-all pack: the columns owned by rank q become the
//                 contiguous block q), 32 x 32 tiles through padded smem,
//                 coalesced on both sides.
//   k_twiddle4  : Y[row][k2] *= W_N^{(row0 + row) k2} (the four-step twiddle,
//                 step (T) of fft_c2.cuh), W_N^x = A[x >> sh] * B[x & mask]
//                 from two fp64-generated tables (x < N, no wrap).
#include <map>
#include <mutex>
#include <utility>

#include "fft_common.cuh"
#include "launch.h"

namespace b200fft {

cudaError_t kernel_setup(const void* kern, int threads, size_t smem, int* grid_max) {
    static std::mutex mu;
    static std::map<std::pair<const void*, int>, int> done;  // (kernel, device) -> persistent grid
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find({kern, dev});
    if (it == done.end()) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int sms = 0, occ = 0;
        if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (e == cudaSuccess && threads > 0)
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem);
        if (e != cudaSuccess) return e;
        it = done.emplace(std::make_pair(kern, dev), sms * (occ > 0 ? occ : 1)).first;
    }
    if (grid_max) *grid_max = it->second;
    return cudaSuccess;
}


namespace {

template <typename T>
__global__ void __launch_bounds__(256) k_transpose(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out,
                                                   int64_t R, int64_t Cn) {
    __shared__ cpx<T> tile[32][33];
    const int64_t mat = blockIdx.z;
    const cpx<T>* src = in + mat * R * Cn;
    cpx<T>* dst = out + mat * R * Cn;
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t r = r0 + ty + i, c = c0 + tx;
        if (r < R && c < Cn) tile[ty + i][tx] = src[r * Cn + c];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t c = c0 + ty + i, r = r0 + tx;
        if (r < R && c < Cn) dst[c * R + r] = tile[tx][ty + i];
    }
}

template <typename T, bool INV>
__global__ void __launch_bounds__(256) k_twiddle4(cpx<T>* __restrict__ y, int64_t rows, int64_t L, int64_t row0,
                                                  const cpx<T>* __restrict__ ta, const cpx<T>* __restrict__ tb,
                                                  int sh) {
    const int64_t total = rows * L;
    const int64_t mask = ((int64_t)1 << sh) - 1;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / L, k2 = i - row * L;
        const int64_t x = (row0 + row) * k2;
        const cpx<T> w = cmul(__ldg(ta + (x >> sh)), __ldg(tb + (x & mask)));
        y[i] = cmul_dir<INV>(y[i], w);
    }
}

// The paper's combine step (Sec. 4): the receiver of a round holds
// E = DFT_M of x[q + 2S j] and gets O = DFT_M of x[q + S + 2S j] from rank
// q + S; one radix-2 level gives the DFT_{2M} of x[q + S j]:
//   Y[k]     = (E[k] + W_{2M}^k O[k]) / 2
//   Y[k + M] = (E[k] - W_{2M}^k O[k]) / 2,   k < M
// (the 1/2 keeps the paper's normalisation: every branch carries its 1/len,
// so l halvings give the 1/n of Eq. E2).  W_{2M}^k = W_n^{k n / (2M)} from the
// two fp64-generated tables (ta[x >> sh] * tb[x & mask]).  `nb` independent
// combines (virtual ranks): E_b = e + b * es, O_b = o + b * es, Y_b = y + b * ys.
template <typename T>
__global__ void __launch_bounds__(256) k_tree_combine(const cpx<T>* __restrict__ e, const cpx<T>* __restrict__ o,
                                                      cpx<T>* __restrict__ y, int64_t M, int64_t nb, int64_t es,
                                                      int64_t ys, int64_t xstep, const cpx<T>* __restrict__ ta,
                                                      const cpx<T>* __restrict__ tb, int sh) {
    const int64_t total = M * nb;
    const int64_t mask = ((int64_t)1 << sh) - 1;
    const T half = (T)0.5;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = i / M, k = i - b * M;
        const int64_t x = k * xstep;
        const cpx<T> w = cmul(__ldg(ta + (x >> sh)), __ldg(tb + (x & mask)));
        const cpx<T> a = e[b * es + k];
        const cpx<T> t = cmul(o[b * es + k], w);
        y[b * ys + k] = cscale(cadd(a, t), half);
        y[b * ys + k + M] = cscale(csub(a, t), half);
    }
}

// Distributed transpose (the fused pack -> all-to-all -> unpack of the
// four-step 1D schedule): the global matrix G[P R][Cn] is held in row slabs
// of R rows by P ranks (src.p[s]), G^T[Cn][P R] is wanted in row slabs of Cb
// rows (dst.p[d]).  A launch covers the global rows [row0, row0 + nrows) and
// columns [col0, col0 + ncols): a rank pushing its own rows into the other
// ranks' slabs (peer stores), a rank pulling its own output rows from the
// other ranks' slabs (peer loads), or all P virtual ranks at once.
// R, Cb: powers of two (shifts rsh, bsh); 32 x 32 tiles through padded smem.
template <typename T>
__global__ void __launch_bounds__(256)
    k_dist_transpose(const __grid_constant__ BlockPtrs src, const __grid_constant__ BlockPtrs dst, int rsh, int64_t Cn,
                     int bsh, int64_t Rg, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols) {
    using C = cpx<T>;
    __shared__ C tile[32][33];
    const int64_t gc0 = col0 + (int64_t)blockIdx.x * 32, gr0 = row0 + (int64_t)blockIdx.y * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
    const int64_t rmask = (1ll << rsh) - 1, bmask = (1ll << bsh) - 1;
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t gr = gr0 + ty + i, gc = gc0 + tx;
        if (gr < row0 + nrows && gc < col0 + ncols)
            tile[ty + i][tx] = reinterpret_cast<const C*>(src.p[gr >> rsh])[(gr & rmask) * Cn + gc];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 32; i += 8) {
        const int64_t gc = gc0 + ty + i, gr = gr0 + tx;
        if (gr < row0 + nrows && gc < col0 + ncols)
            reinterpret_cast<C*>(dst.p[gc >> bsh])[(gc & bmask) * Rg + gr] = tile[tx][ty + i];
    }
    __threadfence_system();  // peer stores, read by other GPUs after the following barrier
}

}  // namespace

cudaError_t launch_dist_transpose(int prec, const BlockPtrs& src, const BlockPtrs& dst, int64_t R, int64_t Cn,
                                  int64_t Cb, int64_t P, int64_t row0, int64_t nrows, int64_t col0, int64_t ncols,
                                  cudaStream_t st) {
    if (nrows <= 0 || ncols <= 0) return cudaSuccess;
    if (P > kMaxBlocks || (R & (R - 1)) || (Cb & (Cb - 1))) return cudaErrorInvalidValue;
    const int rsh = ilog2c((int)R), bsh = ilog2c((int)Cb);
    dim3 grid((unsigned)((ncols + 31) / 32), (unsigned)((nrows + 31) / 32), 1);
    if (prec == 0)
        k_dist_transpose<float><<<grid, 256, 0, st>>>(src, dst, rsh, Cn, bsh, P * R, row0, nrows, col0, ncols);
    else
        k_dist_transpose<double><<<grid, 256, 0, st>>>(src, dst, rsh, Cn, bsh, P * R, row0, nrows, col0, ncols);
    return cudaGetLastError();
}

cudaError_t launch_transpose(int prec, const void* in, void* out, int64_t R, int64_t Cn, int64_t nmat,
                             cudaStream_t st) {
    if (R <= 0 || Cn <= 0 || nmat <= 0) return cudaSuccess;
    dim3 grid((unsigned)((Cn + 31) / 32), (unsigned)((R + 31) / 32), (unsigned)nmat);
    if (prec == 0)
        k_transpose<float><<<grid, 256, 0, st>>>(reinterpret_cast<const float2*>(in), reinterpret_cast<float2*>(out), R,
                                                 Cn);
    else
        k_transpose<double><<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out),
                                                  R, Cn);
    return cudaGetLastError();
}

cudaError_t launch_twiddle4(int prec, bool inv, void* y, int64_t rows, int64_t L, int64_t row0, const void* ta,
                            const void* tb, int sh, cudaStream_t st) {
    const int64_t total = rows * L;
    if (total <= 0) return cudaSuccess;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (prec == 0) {
        if (inv)
            k_twiddle4<float, true><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<float2*>(y), rows, L, row0,
                                                                     reinterpret_cast<const float2*>(ta),
                                                                     reinterpret_cast<const float2*>(tb), sh);
        else
            k_twiddle4<float, false><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<float2*>(y), rows, L, row0,
                                                                      reinterpret_cast<const float2*>(ta),
                                                                      reinterpret_cast<const float2*>(tb), sh);
    } else {
        if (inv)
            k_twiddle4<double, true><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<double2*>(y), rows, L, row0,
                                                                      reinterpret_cast<const double2*>(ta),
                                                                      reinterpret_cast<const double2*>(tb), sh);
        else
            k_twiddle4<double, false><<<(unsigned)blocks, 256, 0, st>>>(reinterpret_cast<double2*>(y), rows, L, row0,
                                                                       reinterpret_cast<const double2*>(ta),
                                                                       reinterpret_cast<const double2*>(tb), sh);
    }
    return cudaGetLastError();
}

cudaError_t launch_tree_combine(int prec, const void* e, const void* o, void* y, int64_t M, int64_t nb, int64_t es,
                                int64_t ys, int64_t xstep, const void* ta, const void* tb, int sh, cudaStream_t st) {
    if (M <= 0 || nb <= 0) return cudaSuccess;
    const int64_t total = M * nb;
    const int64_t want = (total + 255) / 256;
    const unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
    if (prec == 0)
        k_tree_combine<float><<<grid, 256, 0, st>>>(
            reinterpret_cast<const float2*>(e), reinterpret_cast<const float2*>(o), reinterpret_cast<float2*>(y), M,
            nb, es, ys, xstep, reinterpret_cast<const float2*>(ta), reinterpret_cast<const float2*>(tb), sh);
    else
        k_tree_combine<double><<<grid, 256, 0, st>>>(
            reinterpret_cast<const double2*>(e), reinterpret_cast<const double2*>(o), reinterpret_cast<double2*>(y),
            M, nb, es, ys, xstep, reinterpret_cast<const double2*>(ta), reinterpret_cast<const double2*>(tb), sh);
    return cudaGetLastError();
}

}  // namespace b200fft
