// fft_real.cuh -- real-input (R2C) and real-output (C2R) rows on the
// Stockham engine (the paper's images are real).
//
// A real row x of M = 2R values is read as the complex row z[n] = x[2n] +
// i x[2n+1] of R points (the same bytes: no repacking).  With Z = DFT_R(z)
// (unnormalised), E[k] = DFT_R(x_even)[k] and O[k] = DFT_R(x_odd)[k]:
//     E[k] = (Z[k] + conj Z[R - k]) / 2,   O[k] = (Z[k] - conj Z[R - k]) / (2i)
//     X[k] = E[k] + W_M^k O[k],   k = 0 .. R   (Z[R] = Z[0]; W_M = e^{-2 pi i/M})
// the half spectrum of Eq. E2's sum (the other half is X[M - k] = conj X[k]).
// The inverse (Eq. E3, unscaled) of a Hermitian X given by k = 0 .. R:
//     Z'[k] = (X[k] + conj X[R - k]) + i W_M^{-k} (X[k] - conj X[R - k]),  k < R
//     IDFT_R(Z')[n] = f[2n] + i f[2n + 1],   f[j] = sum_{k<M} X[k] e^{+2 pi i jk/M}
// (Im X[0] and Im X[R] do not enter f: they are dropped, as a real signal's
// spectrum has none).  W_M^k comes from an fp64-generated table rtw[k], k < R.
#pragma once
#include "fft_engine.cuh"

namespace b200fft {

// out[row][k] = scale * X[k], k = 0 .. R (row stride ld >= R + 1), in: rows of 2R reals
template <typename T, int R, int E, int W>
__global__ void __launch_bounds__(W*(R / E)) k_rows_r2c(const T* __restrict__ in, cpx<T>* __restrict__ out,
                                                        int64_t batch, T scale, const cpx<T>* __restrict__ tw,
                                                        const cpx<T>* __restrict__ rtw, int64_t ld) {
    using C = cpx<T>;
    using F = LineFFT<T, R, E, false>;
    B200FFT_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int t = tid / F::TPL, lt = tid % F::TPL;
    const int64_t row = (int64_t)blockIdx.x * W + t;
    const bool valid = row < batch;
    C* line = reinterpret_cast<C*>(smem_raw) + t * F::LS;
    C v[E];
    const C* zin = reinterpret_cast<const C*>(in + (valid ? row : 0) * 2 * R);
#pragma unroll
    for (int m = 0; m < E; ++m) v[F::pos_in(m)] = valid ? zin[lt + F::TPL * m] : mk((T)0, (T)0);
    F::run(v, line, lt, tw);
    // Z in natural order (padded) in the line buffer, then each thread pairs
    // its k with R - k
    __syncthreads();
#pragma unroll
    for (int m = 0; m < E; ++m) line[F::bpos(lt, m)] = v[F::pos_out(m)];
    __syncthreads();
    if (!valid) return;
    C* o = out + row * ld;
    const T h = (T)0.5;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k = lt + F::TPL * m;
        const C zk = line[F::bpos(lt, m)];
        const C zr = line[pad16((R - k) & (R - 1))];
        // E = (zk + conj zr) / 2, O = -i (zk - conj zr) / 2
        const C e = mk(h * (zk.x + zr.x), h * (zk.y - zr.y));
        const C od = mk(h * (zk.y + zr.y), -h * (zk.x - zr.x));
        o[k] = cscale(cadd(e, cmul(od, __ldg(rtw + k))), scale);
        if (k == 0) o[R] = mk((e.x - od.x) * scale, (T)0);  // X[R] = E[0] - O[0] (real)
    }
}

// out[row][j] = scale * f[j], j < 2R (real), in: rows of R + 1 bins X[0 .. R] (row stride ld)
template <typename T, int R, int E, int W>
__global__ void __launch_bounds__(W*(R / E)) k_rows_c2r(const cpx<T>* __restrict__ in, T* __restrict__ out,
                                                        int64_t batch, T scale, const cpx<T>* __restrict__ tw,
                                                        const cpx<T>* __restrict__ rtw, int64_t ld) {
    using C = cpx<T>;
    using FI = LineFFT<T, R, E, true>;
    B200FFT_PDL_PROLOGUE();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int tid = threadIdx.x;
    const int t = tid / FI::TPL, lt = tid % FI::TPL;
    const int64_t row = (int64_t)blockIdx.x * W + t;
    const bool valid = row < batch;
    C* line = reinterpret_cast<C*>(smem_raw) + t * FI::LS;
    const C* x = in + (valid ? row : 0) * ld;
    // the row X[0 .. R] into the line buffer (X[R] in the spare last slot)
#pragma unroll
    for (int m = 0; m < E; ++m) line[FI::bpos(lt, m)] = valid ? x[lt + FI::TPL * m] : mk((T)0, (T)0);
    if (lt == 0) line[pad16(R)] = valid ? x[R] : mk((T)0, (T)0);
    __syncthreads();
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k = lt + FI::TPL * m;
        C xk = line[FI::bpos(lt, m)];
        C xr = line[pad16(R - k)];  // k = 0: X[R]
        if (k == 0) {                // Im X[0], Im X[R] do not enter a real signal
            xk.y = (T)0;
            xr.y = (T)0;
        }
        const C a = mk(xk.x + xr.x, xk.y - xr.y);  // X[k] + conj X[R - k]
        const C b = mk(xk.x - xr.x, xk.y + xr.y);  // X[k] - conj X[R - k]
        const C wb = cmulc(b, __ldg(rtw + k));      // W_M^{-k} b
        v[FI::pos_in(m)] = mk(a.x - wb.y, a.y + wb.x);  // a + i wb
    }
    // (the engine's first exchange is preceded by a barrier: every pair has
    // been read before the line buffer is overwritten)
    FI::run(v, line, lt, tw);
    if (!valid) return;
    C* o = reinterpret_cast<C*>(out + row * 2 * R);
#pragma unroll
    for (int m = 0; m < E; ++m) o[lt + FI::TPL * m] = cscale(v[FI::pos_out(m)], scale);
}

}  // namespace b200fft
