// fft_engine.cuh -- the CTA-level Stockham engine and the three kernel
// families of libb200fft (sm_100a).
//
// What is computed: the DFT of Eq. E2 (Sec. 2) and the
// unscaled inverse of Eq. E3 / Sec. 3, by a radix-16
// Stockham autosort (natural order out, no bit-reversal pass) instead of the
// paper's in-place radix-2 tree: the same sums, reassociated.
//
// One "line" = one R-point DFT held by TPL = R/E threads, E values per thread
// in registers.  A step of radix rho with span Ns (product of the radices
// before it) is, for every butterfly j < R/rho with k = j mod Ns:
//     v[r]  = a[j + r R/rho] * W_{Ns rho}^{k r}          (r < rho)
//     b[(j - k) rho + k + q Ns] = sum_r v[r] W_rho^{r q}  (q < rho)
// Steps exchange through shared memory (one padded buffer per line).  At the
// boundary of the engine every thread holds the elements lt + TPL*m, m < E,
// of its line (lt = lane within the line), which is what makes global loads
// and stores coalesced and lets a forward and an inverse transform chain in
// registers (the fused filter pipeline).
#pragma once
#include <cmath>
#include <mutex>
#include <set>

#include "fft_common.cuh"
#include "launch.h"

namespace b200fft {

constexpr int RMAX = 8192;  // largest in-CTA DFT

// W_256^k, k < 256 (fp64-generated on the host, rounded once), in the
// constant cache of every module that includes this header (static: one
// copy per translation unit, uploaded by that unit's launchers through
// w256_upload()).  The step twiddles W_{Ns rho}^{k r} of lines of R <= 256
// points are entries of it (index k r 256 / (Ns rho)); in the task-pipeline
// kernels the butterfly index k is uniform (or takes two values) across a
// warp, so these loads are constant-cache broadcasts that take the twiddle
// products off the FP32 pipe (round 2: C2 -3.2%, and more accurate than the
// recurrence's powers).
static __constant__ float2 c_w256[256];

// upload c_w256 for the current device (once per device per module)
static inline cudaError_t w256_upload() {
    static std::mutex mu;
    static std::set<int> done;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    if (done.count(dev)) return cudaSuccess;
    float2 h[256];
    for (int k = 0; k < 256; ++k) {
        const double a = -2.0 * 3.14159265358979323846 * (double)k / 256.0;
        h[k] = make_float2((float)cos(a), (float)sin(a));
    }
    e = cudaMemcpyToSymbol(c_w256, h, sizeof(h));
    if (e == cudaSuccess) done.insert(dev);
    return e;
}
// Twiddles of the in-CTA steps come from the step-major tables of
// fft_common.cuh (tw_base / tw_off), fp64-generated on the host and rounded
// once; kernels receive the pointer to their R's table.

// unpadded smem layout (LAYOUT 1): XOR the low 4 index bits with bits 4..7,
// a permutation inside every 16-element group that makes both the
// consecutive and the stride-16 access patterns of the steps conflict-free
__device__ __forceinline__ int swz16(int i) { return i ^ ((i >> 4) & 15); }
// LAYOUT 2: 16 lines interleaved element by element (element x of line t at
// x * 16 + t: a dense [R][16] TMA box of 16 columns); with the 16 lines as
// the thread-fastest index every exchange is conflict-free

// LAYOUT 5: 64 lines interleaved element by element (element x of line t at
// x * 64 + t: a dense [R][64] TMA box), lines the thread-fastest index
// LAYOUT 3: one warp per 256-point line, E = 8 (steps 8, 8, 4): XOR the low
// 4 index bits with g(bits 4..7), g(c) = c ^ (bit 2 of c) << 3 -- every
// exchange of that schedule hits 16 distinct 8-B bank pairs per half-warp
__device__ __forceinline__ int swz8(int i) {
    const int c = (i >> 4) & 15;
    return i ^ (c ^ (((c >> 2) & 1) << 3));
}
// LAYOUT 4: 8 lines interleaved element by element (element x of line t at
// h(x) * 8 + t, h(x) = x ^ bit 3 of x: a dense [R][8] TMA box of 8 columns
// after the first read) with the 8 lines as the thread-fastest index: the two
// element positions of a half-warp always differ in h's parity
__device__ __forceinline__ int il8(int i) { return (i ^ ((i >> 3) & 1)) * 8; }

// PF: prefetch each step's twiddles into registers before its exchange
// barriers (for kernels with a 128-register budget)
// TWREC: a step's twiddles W^{k r}, r = 1..rho-1, as powers of the one
// table entry W^{k} (rho - 2 complex products, ~rho ulp in fp32) instead of
// rho - 1 loads -- for kernels whose warps are short of load bandwidth.
// TWREC = 2 (complex64, R <= 256): from the constant table c_w256, for
// kernels whose butterfly index is (nearly) uniform across a warp.
// MLX: the largest radix 2^MLX (0: ml_of(E); 5: radix-32 steps for E >= 32)
template <typename T, int R, int E, bool INV, int LAYOUT = 0, bool PF = false, int TWREC = (sizeof(T) == 4),
          int MLX = 0>
struct LineFFT {
    using C = cpx<T>;
    static constexpr int ML = MLX ? MLX : ml_of(E);  // largest radix 2^ML (16, or 8 when E = 8; 32 with MLX 5)
    static constexpr int TPL = R / E;
    static constexpr int S = n_steps(R, ML);
    static constexpr int LS = pad16c(R) + 1;  // odd line stride in smem (slots)
    static constexpr int RHO0 = radix_at(R, 0, ML);
    static constexpr int RHOL = radix_at(R, S - 1, ML);
    static_assert(E % RHO0 == 0 && E % RHOL == 0, "E must be a multiple of every radix");

    // register slot of boundary element m (element index lt + TPL m)
    __device__ static constexpr int pos_in(int m) {
        return (m % (E / RHO0)) * RHO0 + m / (E / RHO0);
    }
    __device__ static constexpr int pos_out(int m) {
        return (m % (E / RHOL)) * RHOL + m / (E / RHOL);
    }

    template <int s>
    __device__ __forceinline__ static void compute(C* v, int lt, const C* __restrict__ tw) {
        constexpr int rho = radix_at(R, s, ML), Ns = span_at(R, s, ML), nb = E / rho;
#pragma unroll
        for (int b = 0; b < nb; ++b) {
            if constexpr (Ns > 1) {
                const int j = lt + b * TPL;
                const int k = j & (Ns - 1);
                const C* __restrict__ ts = tw + tw_off(R, s, ML) + k;
                if constexpr (TWREC == 2) {
                    static_assert(sizeof(T) == 4 && 256 % (Ns * rho) == 0, "constant twiddles: R <= 256, complex64");
                    constexpr int SC = 256 / (Ns * rho);
#pragma unroll
                    for (int r = 1; r < rho; ++r)
                        v[b * rho + r] = cmul_dir<INV>(v[b * rho + r], c_w256[(k * r * SC) & 255]);
                } else if constexpr (TWREC) {
                    const C w1 = __ldg(ts);
                    C w = w1;
#pragma unroll
                    for (int r = 1; r < rho; ++r) {
                        v[b * rho + r] = cmul_dir<INV>(v[b * rho + r], w);
                        if (r + 1 < rho) w = cmul(w, w1);
                    }
                } else {
#pragma unroll
                    for (int r = 1; r < rho; ++r) {
                        const C w = __ldg(ts + (r - 1) * Ns);
                        v[b * rho + r] = cmul_dir<INV>(v[b * rho + r], w);
                    }
                }
            }
            dft<rho, INV>(v + b * rho);
        }
    }

    // Twiddles of step s prefetched into registers (issued before the
    // exchange barriers of the step, so their latency hides behind them) when
    // they are few enough: (rho - 1) * nb <= 16 complex values.
    template <int s>
    static constexpr int ntw() {
        return (span_at(R, s, ML) > 1) ? (radix_at(R, s, ML) - 1) * (E / radix_at(R, s, ML)) : 0;
    }
    template <int s>
    static constexpr bool prefetch_tw() {
        return PF && !TWREC && ntw<s>() > 0 && ntw<s>() <= 16;
    }
    template <int s>
    __device__ __forceinline__ static void load_tw(C* w, int lt, const C* __restrict__ tw) {
        constexpr int rho = radix_at(R, s, ML), Ns = span_at(R, s, ML), nb = E / rho;
#pragma unroll
        for (int b = 0; b < nb; ++b) {
            const int k = (lt + b * TPL) & (Ns - 1);
            const C* __restrict__ ts = tw + tw_off(R, s, ML) + k;
#pragma unroll
            for (int r = 1; r < rho; ++r) w[b * (rho - 1) + r - 1] = __ldg(ts + (r - 1) * Ns);
        }
    }
    template <int s>
    __device__ __forceinline__ static void compute_tw(C* v, const C* w) {
        constexpr int rho = radix_at(R, s, ML), nb = E / rho;
#pragma unroll
        for (int b = 0; b < nb; ++b) {
#pragma unroll
            for (int r = 1; r < rho; ++r) v[b * rho + r] = cmul_dir<INV>(v[b * rho + r], w[b * (rho - 1) + r - 1]);
            dft<rho, INV>(v + b * rho);
        }
    }

    // Padded smem indices.  pad16(x + c) = pad16(x) + c + c/16 whenever c is a
    // multiple of 16, so one pad16 per butterfly and compile-time offsets
    // (folded into the LDS/STS immediates) cover every element.
    template <int s>
    __device__ __forceinline__ static void write_out(C* line, const C* v, int lt) {
        constexpr int rho = radix_at(R, s, ML), Ns = span_at(R, s, ML), nb = E / rho;
#pragma unroll
        for (int b = 0; b < nb; ++b) {
            const int j = lt + b * TPL;
            const int k = j & (Ns - 1);
            const int base = (j - k) * rho + k;
            if constexpr (LAYOUT == 1) {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[swz16(base + q * Ns)] = v[b * rho + q];
            } else if constexpr (LAYOUT == 2) {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[(base + q * Ns) * 16] = v[b * rho + q];
            } else if constexpr (LAYOUT == 5) {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[(base + q * Ns) * 64] = v[b * rho + q];
            } else if constexpr (LAYOUT == 3) {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[swz8(base + q * Ns)] = v[b * rho + q];
            } else if constexpr (LAYOUT == 4) {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[il8(base + q * Ns)] = v[b * rho + q];

            } else if constexpr (Ns % 16 == 0) {
                const int pb = pad16(base);
#pragma unroll
                for (int q = 0; q < rho; ++q) line[pb + q * (Ns + Ns / 16)] = v[b * rho + q];
            } else if constexpr (Ns == 1 && rho == 16) {
                const int pb = 17 * j;  // base = 16 j: pad16(16 j + q) = 17 j + q
#pragma unroll
                for (int q = 0; q < rho; ++q) line[pb + q] = v[b * rho + q];
            } else {
#pragma unroll
                for (int q = 0; q < rho; ++q) line[pad16(base + q * Ns)] = v[b * rho + q];
            }
        }
    }

    template <int s>
    __device__ __forceinline__ static void read_in(const C* line, C* v, int lt) {
        constexpr int rho = radix_at(R, s, ML), nb = E / rho;
        constexpr int st = R / rho;
#pragma unroll
        for (int b = 0; b < nb; ++b) {
            const int j = lt + b * TPL;
            if constexpr (LAYOUT == 1) {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[swz16(j + r * st)];
            } else if constexpr (LAYOUT == 2) {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[(j + r * st) * 16];
            } else if constexpr (LAYOUT == 5) {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[(j + r * st) * 64];
            } else if constexpr (LAYOUT == 3) {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[swz8(j + r * st)];
            } else if constexpr (LAYOUT == 4) {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[il8(j + r * st)];

            } else if constexpr (st % 16 == 0) {
                const int pj = pad16(j);
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[pj + r * (st + st / 16)];
            } else {
#pragma unroll
                for (int r = 0; r < rho; ++r) v[b * rho + r] = line[pad16(j + r * st)];
            }
        }
    }

    // padded index of boundary element m (element lt + TPL m of the line)
    __device__ __forceinline__ static int bpos(int lt, int m) {
        if constexpr (LAYOUT == 1) return swz16(lt + TPL * m);
        else if constexpr (LAYOUT == 2) return (lt + TPL * m) * 16;
        else if constexpr (LAYOUT == 5) return (lt + TPL * m) * 64;
        else if constexpr (LAYOUT == 3) return swz8(lt + TPL * m);
        else if constexpr (LAYOUT == 4) return il8(lt + TPL * m);
        else if constexpr (TPL % 16 == 0) return pad16(lt) + m * (TPL + TPL / 16);
        else return pad16(lt + TPL * m);
    }

    // Barrier between steps: the whole CTA, or (bar >= 1) only the TPL
    // threads of this line through named barrier `bar` -- lines of one CTA
    // then never wait for each other.  Needs TPL % 32 == 0 (whole warps).
    __device__ __forceinline__ static void lsync(int bar) {
        if constexpr (TPL == 32) {
            if (bar == -32) {  // a line owned by one warp
                __syncwarp();
                return;
            }
        }
        if (bar < 0) {  // the -bar threads of a warp-specialised CTA's compute group (named barrier 1)
            asm volatile("bar.sync 1, %0;\n" ::"r"(-bar) : "memory");
            return;
        }
        if constexpr (TPL % 32 == 0) {
            if (bar > 0) {
                asm volatile("bar.sync %0, %1;\n" ::"r"(bar), "n"(TPL) : "memory");
                return;
            }
        }
        __syncthreads();
    }

    template <int s>
    __device__ __forceinline__ static void run_from(C* v, C* line, int lt, const C* __restrict__ tw, int bar) {
        if constexpr (s < S) {
            if constexpr (prefetch_tw<s>()) {
                C w[ntw<s>()];
                load_tw<s>(w, lt, tw);
                lsync(bar);
                write_out<s - 1>(line, v, lt);
                lsync(bar);
                read_in<s>(line, v, lt);
                compute_tw<s>(v, w);
            } else {
                lsync(bar);
                write_out<s - 1>(line, v, lt);
                lsync(bar);
                read_in<s>(line, v, lt);
                compute<s>(v, lt, tw);
            }
            run_from<s + 1>(v, line, lt, tw, bar);
        }
    }

    // v holds the step-0 inputs (pos_in layout) -> v holds the outputs (pos_out layout)
    __device__ __forceinline__ static void run(C* v, C* line, int lt, const C* __restrict__ tw, int bar = 0) {
        compute<0>(v, lt, tw);
        run_from<1>(v, line, lt, tw, bar);
    }
};

// --------------------------------------------------------------------------
// Kernel family A: contiguous rows, one whole transform per line.
//   out[row][i] = scale * sum_j in[row][j] W_R^{+-ij},  rows < batch.
// W lines (rows) per CTA.  REAL_IN: input rows are float32 real values
// (promotion to complex fused into the load, BASELINE configs[2]).
// in_sh / out_sh >= 0: the rows are stored in column blocks of 2^sh (the
// all-to-all layout of the slab-decomposed 2D transform):
// element (row, v) at ((C*)blocks.p[v >> sh])[(row << sh) | (v & (2^sh - 1))],
// the blocks local or in peer memory (launch.h BlockPtrs).
// --------------------------------------------------------------------------
__device__ __forceinline__ int64_t block_index(int64_t row, int v, int sh) {
    return (row << sh) | (int64_t)(v & ((1 << sh) - 1));
}

// FILT: a row filter pass of the separable pipeline: forward
// transform -> * rowfilt[v] * scale -> inverse transform, stored unscaled.
template <typename T, int R, int E, bool FILT, int LAYOUT = 0, bool PF = false, int TWREC = 0, int MLX = 0>
__device__ __forceinline__ void row_filter_pass(cpx<T>* v, cpx<T>* line, int lt, const cpx<T>* __restrict__ tw,
                                                const T* __restrict__ rowfilt, T& scale, int bar = 0) {
    if constexpr (FILT) {
        using F = LineFFT<T, R, E, false, LAYOUT, PF, TWREC, MLX>;
        using FI = LineFFT<T, R, E, true, LAYOUT, PF, TWREC, MLX>;
        cpx<T> w[E];
#pragma unroll
        for (int m = 0; m < E; ++m)
            w[FI::pos_in(m)] = cscale(v[F::pos_out(m)], __ldg(rowfilt + lt + F::TPL * m) * scale);
        FI::run(w, line, lt, tw, bar);
#pragma unroll
        for (int m = 0; m < E; ++m) v[F::pos_out(m)] = w[FI::pos_out(m)];
        scale = (T)1;
    }
}

template <typename T, int R, int E, int W, bool INV, bool REAL_IN, bool FILT = false>
__global__ void __launch_bounds__(W*(R / E)) k_rows(const void* __restrict__ in_, cpx<T>* __restrict__ out,
                                                    int64_t batch, T scale, const cpx<T>* __restrict__ tw,
                                                    int in_sh, int out_sh, const T* __restrict__ rowfilt,
                                                    const __grid_constant__ BlockPtrs ib,
                                                    const __grid_constant__ BlockPtrs ob) {
    using C = cpx<T>;
    using F = LineFFT<T, R, E, INV>;
    B200FFT_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* smem = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int64_t row = (int64_t)blockIdx.x * W + t;
    const bool valid = row < batch;
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = mk((T)0, (T)0);
    if (valid) {
        if (in_sh < 0) {  // natural rows: one base address, compile-time offsets
            const int64_t base = row * R + lt;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                if constexpr (REAL_IN)
                    v[F::pos_in(m)] = mk((T)__ldg(reinterpret_cast<const float*>(in_) + base + F::TPL * m), (T)0);
                else
                    v[F::pos_in(m)] = reinterpret_cast<const C*>(in_)[base + F::TPL * m];
            }
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int x = lt + F::TPL * m;
                const int64_t idx = block_index(row, x, in_sh);
                if constexpr (REAL_IN)
                    v[F::pos_in(m)] = mk((T)reinterpret_cast<const float*>(ib.p[x >> in_sh])[idx], (T)0);
                else
                    v[F::pos_in(m)] = reinterpret_cast<const C*>(ib.p[x >> in_sh])[idx];
            }
        }
    }
    F::run(v, smem + t * F::LS, lt, tw);
    row_filter_pass<T, R, E, FILT>(v, smem + t * F::LS, lt, tw, rowfilt, scale);
    if (valid) {
        if (out_sh < 0) {
            C* o = out + row * R + lt;
#pragma unroll
            for (int m = 0; m < E; ++m) o[F::TPL * m] = cscale(v[F::pos_out(m)], scale);
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int x = lt + F::TPL * m;
                reinterpret_cast<C*>(ob.p[x >> out_sh])[block_index(row, x, out_sh)] =
                    cscale(v[F::pos_out(m)], scale);
            }
            // the blocks may be peer memory read by other GPUs after the
            // stream-ordered barrier that follows this kernel
            __threadfence_system();
        }
    }
}

// --------------------------------------------------------------------------
// Filters of the 2D pipeline (Sec. 6), evaluated per (u, v):
//   GAUSS: g_u[u] * g_v[v] (separable fp64-generated 1D tables, b200fft.h)
//   IDEAL_LITERAL: 0 if (u-N/2)^2 + (v-M/2)^2 <= b^2 else 1   (Eq. filtro)
//   IDEAL_LOWPASS: 1 if k_u^2 + k_v^2 <= b^2 else 0 (signed k)
// --------------------------------------------------------------------------
struct FilterArgs {
    int kind;           // fft_filter
    double b2;          // radius^2 for the ideal filters
    const void* gu;     // T[N] (GAUSS)
    const void* gv;     // T[M] (GAUSS)
    int64_t N, M;       // global grid
    int64_t col_off;    // global index of local column 0 (column slab of a distributed plan)
    float* spec;        // optional (MODE 2, complex64): |F(u,v)| * spec_scale -> spec[img][u][v]
    float spec_scale;   // eq5's 1/N (the column pass holds the unnormalised 2D sums)
    // four-step column passes (k_cols_pipe MODE 3 / 4, kind 6): twiddle
    // W_L^{(col / tdiv) * u} from tw_l (L entries, fp64-generated), and the
    // pass-B filter index img + n1 * u into gu
    const void* tw_l;
    int64_t tdiv;
    int64_t n1;
};

// pass-B filter of the four-step column passes: g_N[k1 + n1 k2] (kind 6,
// the column factor of the separable Gaussian) or, kind 7 (the distributed
// column slab, whose row passes are unfiltered), times g_M[col + col_off]
template <typename T>
__device__ __forceinline__ T fourstep_filter(const FilterArgs& f, int64_t img, int64_t u, int64_t col) {
    T h = __ldg(reinterpret_cast<const T*>(f.gu) + img + f.n1 * u);
    if (f.kind == 7) h *= __ldg(reinterpret_cast<const T*>(f.gv) + col + f.col_off);
    return h;
}

// spectrum sqrt(Re^2 + Im^2) of one forward-transformed column (Sec. 6,
// P:369-373), written when the pipeline's caller asked for it
template <typename C>
__device__ __forceinline__ float spec_mag(C a, float s) {
    const float x = (float)a.x, y = (float)a.y;
    return sqrtf(fmaf(x, x, y * y)) * s;
}

template <typename T>
__device__ __forceinline__ T filter_value(const FilterArgs& f, int64_t u, int64_t v) {
    if (f.kind == 1) {
        return __ldg(reinterpret_cast<const T*>(f.gu) + u) * __ldg(reinterpret_cast<const T*>(f.gv) + v);
    } else if (f.kind == 2) {
        const double du = (double)(u - f.N / 2), dv = (double)(v - f.M / 2);
        return (du * du + dv * dv <= f.b2) ? (T)0 : (T)1;
    } else if (f.kind == 3) {
        const double ku = (double)(u < f.N / 2 ? u : u - f.N), kv = (double)(v < f.M / 2 ? v : v - f.M);
        return (ku * ku + kv * kv <= f.b2) ? (T)1 : (T)0;
    } else if (f.kind == 5) {  // column factor of a separable filter (the row factor ran in k_rows)
        return __ldg(reinterpret_cast<const T*>(f.gu) + u);
    }
    return (T)1;
}

// --------------------------------------------------------------------------
// Kernel family B: columns of [img][R][S] (R rows of S complex), W adjacent
// columns per CTA (coalesced W-element row segments, staged through smem).
//   MODE 0: forward column DFT, times scale
//   MODE 1: inverse column DFT, times scale
//   MODE 2: forward -> * H(u, v) * scale -> inverse (the fused middle of the
//           2D filter pipeline; scale = 1/(N M))
// --------------------------------------------------------------------------
// smem line stride of the column tiles: a multiple of the 128-B bank row plus
// 128 B / (W * elem) so that the W-wide staging rows hit distinct banks
template <typename T, int R, int W>
__host__ __device__ constexpr int cols_ls() {
    constexpr int SL = 128 / (int)sizeof(cpx<T>);
    return ((pad16c(R) + SL - 1) / SL) * SL + (W >= SL ? 1 : SL / W);
}

// MINB > 0: a register cap for MINB CTAs/SM (0: the compiler's choice)
template <typename T, int R, int E, int W, int MODE, int MINB = 0>
__global__ void __launch_bounds__(W*(R / E), MINB) k_cols(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out,
                                                    int64_t S, T scale, const cpx<T>* __restrict__ tw,
                                                    FilterArgs filt) {
    using C = cpx<T>;
    B200FFT_PDL_PROLOGUE();
    // MODE 3 / 4 / kind 6: the four-step column passes (see k_cols_pipe)
    constexpr bool INV0 = (MODE == 1 || MODE == 4);
    using F = LineFFT<T, R, E, INV0>;
    using FI = LineFFT<T, R, E, true>;
    constexpr int NT = W * F::TPL;
    constexpr int LSC = cols_ls<T, R, W>();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* smem = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    // short lines (TPL < 32): lines are the thread-fastest index, so a warp
    // touches 32 different lines at one offset and the odd line stride keeps
    // every exchange conflict-free (lane-fastest within a 4-/8-/16-thread line
    // put several lines in one bank group: 4-way conflicts, profiles/README.md)
    constexpr bool LF = F::TPL < 32;
    const int t = LF ? tid % W : tid / F::TPL, lt = LF ? tid / W : tid % F::TPL;
    const int64_t s0 = (int64_t)blockIdx.x * W;
    const int64_t img = blockIdx.y;
    const C* src = in + img * (int64_t)R * S + s0;
    C* dst = out + img * (int64_t)R * S + s0;
    const int wv = (int)((S - s0) < W ? (S - s0) : W);  // ragged last tile

    // fully unrolled so that all of a thread's loads are in flight at once
#pragma unroll
    for (int it = 0; it < (W * R) / NT; ++it) {
        const int idx = tid + it * NT;
        const int tt = idx % W, r = idx / W;
        smem[tt * LSC + pad16(r)] = (tt < wv) ? src[(int64_t)r * S + tt] : mk((T)0, (T)0);
    }
    __syncthreads();
    C* line = smem + t * LSC;
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
    if constexpr (MODE == 4) {  // conj(W^{n2 (lt + TPL m)}) by recurrence
        const int64_t n2 = (s0 + t) / filt.tdiv;
        const C* tl = reinterpret_cast<const C*>(filt.tw_l);
        C wm = __ldg(tl + n2 * lt);
        const C ws = __ldg(tl + n2 * F::TPL);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            v[F::pos_in(m)] = cmulc(v[F::pos_in(m)], wm);
            wm = cmul(wm, ws);
        }
    }
    // lines synchronise on their own named barrier (1 + t) between steps
    const int bar = (!LF && F::TPL % 32 == 0 && W <= 15) ? 1 + t : 0;
    F::run(v, line, lt, tw, bar);
    if constexpr (MODE == 3) {  // W^{n2 (lt + TPL m)} by recurrence
        const int64_t n2 = (s0 + t) / filt.tdiv;
        const C* tl = reinterpret_cast<const C*>(filt.tw_l);
        C wm = __ldg(tl + n2 * lt);
        const C ws = __ldg(tl + n2 * F::TPL);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            v[F::pos_out(m)] = cmul(v[F::pos_out(m)], wm);
            wm = cmul(wm, ws);
        }
    }
    if constexpr (MODE == 2) {
        C w[E];
        const int64_t col = s0 + t;
        if (filt.spec != nullptr && col < S) {
            float* sp = filt.spec + img * (int64_t)R * S + col;
#pragma unroll
            for (int m = 0; m < E; ++m) sp[(int64_t)(lt + F::TPL * m) * S] = spec_mag(v[F::pos_out(m)], filt.spec_scale);
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int64_t u = lt + F::TPL * m;
            const T hv = (filt.kind >= 6) ? fourstep_filter<T>(filt, img, u, col < S ? col : 0)
                                          : filter_value<T>(filt, u, col + filt.col_off);
            const T h = (col < S) ? hv * scale : (T)0;
            w[FI::pos_in(m)] = cscale(v[F::pos_out(m)], h);
        }
        FI::run(w, line, lt, tw, bar);
        F::lsync(bar);
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = w[FI::pos_out(m)];
    } else {
        F::lsync(bar);
#pragma unroll
        for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
    }
    __syncthreads();
    // fully unrolled so that all of a thread's loads are in flight at once
#pragma unroll
    for (int it = 0; it < (W * R) / NT; ++it) {
        const int idx = tid + it * NT;
        const int tt = idx % W, r = idx / W;
        if (tt < wv) dst[(int64_t)r * S + tt] = smem[tt * LSC + pad16(r)];
    }
}

// --------------------------------------------------------------------------
// Kernel family C: one global Stockham pass of radix R over rows of length L
// (multi-pass transforms, L > RMAX), W adjacent butterflies j per CTA:
//   v[r] = a[j + r L/R] * W_{Ns R}^{k r},  k = j mod Ns
//   b[(j - k) R + k + q Ns] = scale * sum_r v[r] W_R^{r q}
// The pass twiddle W_{Ns R}^{k r} comes from two fp64-generated tables laid
// out [r][k] so that adjacent lines (adjacent k) read adjacent entries:
//   pa[r KLO + (k mod KLO)] * pb[r (Ns/KLO) + k / KLO]   (pb only if Ns > KLO)
// --------------------------------------------------------------------------
template <typename T, int R, int E, int W, bool INV>
__global__ void __launch_bounds__(W*(R / E)) k_pass(const cpx<T>* __restrict__ in, cpx<T>* __restrict__ out,
                                                    int64_t L, int64_t Ns, int64_t nlines, T scale,
                                                    const cpx<T>* __restrict__ tw,
                                                    const cpx<T>* __restrict__ pa,
                                                    const cpx<T>* __restrict__ pb, int klo_sh) {
    using C = cpx<T>;
    // complex64: step twiddles as powers of one table entry (TWREC) and the
    // pass twiddles W^{k (r0 + it RS)} = W^{k r0} (W^{k RS})^it from two table
    // products per thread -- fewer loads per element (fp32, ~R / RS ulp)
    constexpr bool REC = sizeof(T) == 4;
    using F = LineFFT<T, R, E, INV, 0, false, REC>;
    constexpr int NT = W * F::TPL;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* smem = reinterpret_cast<C*>(smem_raw);
    const int tid = threadIdx.x;
    // short lines (TPL < 32): lines are the thread-fastest index, so a warp
    // touches 32 different lines at one offset and the odd line stride keeps
    // every exchange conflict-free (lane-fastest within a 4-/8-/16-thread line
    // put several lines in one bank group: 4-way conflicts, profiles/README.md)
    constexpr bool LF = F::TPL < 32;
    const int t = LF ? tid % W : tid / F::TPL, lt = LF ? tid / W : tid % F::TPL;
    const int64_t LR = L / R;                     // butterflies per transform
    const int64_t gl0 = (int64_t)blockIdx.x * W;  // first line of the tile (W | LR)
    const int64_t bidx = gl0 / LR;
    const int64_t j0 = gl0 - bidx * LR;
    const C* src = in + bidx * L;
    C* dst = out + bidx * L;
    const int64_t KLO = (int64_t)1 << klo_sh;
    const int64_t nhi = Ns >> klo_sh;
    // Thread tid always handles tile line tt = tid % W and elements
    // r = tid / W + it * RS (RS = NT / W = TPL, a multiple of 16 for R >= 256):
    // one base address per thread and constant strides per iteration.
    constexpr int RS = NT / W;
    static_assert(NT % W == 0, "tile shape");
    const int tt = tid % W, r0 = tid / W;
    const int64_t jt = j0 + tt;
    const int64_t kt = jt & (Ns - 1);
    {
        const C* s = src + jt + (int64_t)r0 * LR;
        const int64_t sstep = (int64_t)RS * LR;
        const C* wa = pa + (int64_t)r0 * KLO + (kt & (KLO - 1));
        const C* wb = pb + (int64_t)r0 * nhi + (kt >> klo_sh);
        C* d = smem + tt * F::LS;
        const int pr0 = pad16(r0);
        C w = mk((T)1, (T)0), wstep = w;
        if (REC && Ns > 1) {  // W^{k r0} and W^{k RS}
            w = __ldg(wa);
            if (nhi > 1) w = cmul(w, __ldg(wb));
            const int64_t drs = (int64_t)RS;
            wstep = __ldg(pa + drs * KLO + (kt & (KLO - 1)));
            if (nhi > 1) wstep = cmul(wstep, __ldg(pb + drs * nhi + (kt >> klo_sh)));
        }
        // fully unrolled so that all of a thread's loads are in flight at once
#pragma unroll
        for (int it = 0; it < (W * R) / NT; ++it) {
            C a = s[it * sstep];
            if (Ns > 1) {
                if constexpr (REC) {
                    a = cmul_dir<INV>(a, w);
                    w = cmul(w, wstep);
                } else {
                    C wl = __ldg(wa + (int64_t)it * RS * KLO);
                    if (nhi > 1) wl = cmul(wl, __ldg(wb + (int64_t)it * RS * nhi));
                    a = cmul_dir<INV>(a, wl);
                }
            }
            d[(RS % 16 == 0) ? pr0 + it * (RS + RS / 16) : pad16(r0 + it * RS)] = a;
        }
    }
    __syncthreads();
    C* line = smem + t * F::LS;
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[F::pos_in(m)] = line[F::bpos(lt, m)];
    F::run(v, line, lt, tw);
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = cscale(v[F::pos_out(m)], scale);
    __syncthreads();
    if (Ns >= W) {  // consecutive threads -> consecutive k: W-element runs per q
        C* d = dst + (jt - kt) * R + kt + (int64_t)r0 * Ns;
        const C* sm = smem + tt * F::LS;
        const int pq0 = pad16(r0);
#pragma unroll
        for (int it = 0; it < (W * R) / NT; ++it)
            d[(int64_t)it * RS * Ns] = sm[(RS % 16 == 0) ? pq0 + it * (RS + RS / 16) : pad16(r0 + it * RS)];
    } else {  // Ns == 1: the tile's output is one contiguous block of W R elements
#pragma unroll
        for (int it = 0; it < (W * R) / NT; ++it) {
            const int idx = tid + it * NT;
            const int q = idx % R, tl = idx / R;
            const int64_t j = j0 + tl, k = j & (Ns - 1);
            dst[(j - k) * R + k + (int64_t)q * Ns] = smem[tl * F::LS + pad16(q)];
        }
    }
}

}  // namespace b200fft
