// fft_common.cuh -- complex arithmetic and in-register DFT butterflies for the
// sm_100a kernels of libb200fft.
//
// The transforms computed are the paper's DFT (Eq. E2) and
// its unscaled inverse (Eq. E3 / Sec. 3).  Here only the
// building blocks live: a radix-rho DFT on values held in registers,
//     V[q] = sum_{r<rho} v[r] * w^(r q),  w = exp(-+2 pi i / rho),
// with compile-time constant twiddles.  The minus sign is the forward
// transform (INV = false), the plus sign the inverse (INV = true).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace b200fft {

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while the
// previous kernel on its stream is finishing; it waits here, before its first
// global-memory access, for that kernel's results, and lets the next kernel
// launch early.  Both instructions are no-ops for an ordinary launch.
#define B200FFT_PDL_PROLOGUE()                                     \
    do {                                                           \
        asm volatile("griddepcontrol.wait;\n" ::: "memory");       \
        asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); \
    } while (0)

template <typename T> struct cpx_t;
template <> struct cpx_t<float> { using type = float2; };
template <> struct cpx_t<double> { using type = double2; };
template <typename T> using cpx = typename cpx_t<T>::type;

__device__ __forceinline__ float2 mk(float x, float y) { return make_float2(x, y); }
__device__ __forceinline__ double2 mk(double x, double y) { return make_double2(x, y); }

template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return mk(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return mk(a.x - b.x, a.y - b.y); }
// a * b
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
    return mk(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename C, typename S> __device__ __forceinline__ C cscale(C a, S s) {
    return mk(a.x * s, a.y * s);
}

// complex64 specialisations on the sm_100 packed-fp32 pipe (add/sub/mul/fma
// .f32x2 -> FADD2 / FMUL2 / FFMA2): one instruction per complex add, two per
// complex multiply (ptxas folds the (y, x) swap and the one-sided negation
// into the FFMA2 operand modifiers), half the issue slots of scalar fp32.
// Rounding is the same as the scalar code (RN, FMA contraction).
__device__ __forceinline__ uint64_t pk2(float2 a) {
    uint64_t r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 up2(uint64_t r) {
    float2 v;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
    return v;
}
__device__ __forceinline__ float2 cadd(float2 a, float2 b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return up2(r);
}
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    uint64_t r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return up2(r);
}
// a * w = (a.x, a.y) * (w.x, w.x) + (a.y, a.x) * (-w.y, w.y)
__device__ __forceinline__ float2 cmul(float2 a, float2 w) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(make_float2(w.x, w.x))));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(pk2(make_float2(a.y, a.x))), "l"(pk2(make_float2(-w.y, w.y))));
    return up2(r);
}
// a * conj(w) = (a.x, a.y) * (w.x, w.x) + (a.y, a.x) * (w.y, -w.y)
__device__ __forceinline__ float2 cmulc(float2 a, float2 w) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(make_float2(w.x, w.x))));
    asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(r) : "l"(pk2(make_float2(a.y, a.x))), "l"(pk2(make_float2(w.y, -w.y))));
    return up2(r);
}
__device__ __forceinline__ float2 cscale(float2 a, float s) {
    uint64_t r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(make_float2(s, s))));
    return up2(r);
}

template <bool CONJ, typename C> __device__ __forceinline__ C cmul_dir(C a, C b) {
    if constexpr (CONJ) return cmulc(a, b);
    else return cmul(a, b);
}
// -i * a (forward quarter turn) / +i * a (inverse)
template <bool INV, typename C> __device__ __forceinline__ C rot_quarter(C a) {
    if constexpr (INV) return mk(-a.y, a.x);
    else return mk(a.y, -a.x);
}

// cos / sin of 2 pi e / 16 (exact decimal expansions, 20 digits)
__host__ __device__ constexpr double cos16(int e) {
    switch (e & 15) {
        case 0: return 1.0;
        case 1: return 0.92387953251128675613;
        case 2: return 0.70710678118654752440;
        case 3: return 0.38268343236508977173;
        case 4: return 0.0;
        case 5: return -0.38268343236508977173;
        case 6: return -0.70710678118654752440;
        case 7: return -0.92387953251128675613;
        case 8: return -1.0;
        case 9: return -0.92387953251128675613;
        case 10: return -0.70710678118654752440;
        case 11: return -0.38268343236508977173;
        case 12: return 0.0;
        case 13: return 0.38268343236508977173;
        case 14: return 0.70710678118654752440;
        default: return 0.92387953251128675613;
    }
}
__host__ __device__ constexpr double sin16(int e) { return cos16(e - 4); }  // sin x = cos(x - pi/2)
// cos of 2 pi e / 32: even e from cos16, odd e from the first-octant values
// (exact decimal expansions, 20 digits) by the quadrant symmetries
__host__ __device__ constexpr double cos32(int e) {
    e &= 31;
    if (!(e & 1)) return cos16(e / 2);
    // cos(2 pi e / 32) for e = 1, 3, 5, 7 (and 9..15 = -cos of 16 - e)
    const int q = e < 16 ? e : 32 - e;  // cos is even: fold to e <= 16
    switch (q) {
        case 1: return 0.98078528040323044913;
        case 3: return 0.83146961230254523708;
        case 5: return 0.55557023301960222474;
        case 7: return 0.19509032201612826785;
        case 9: return -0.19509032201612826785;
        case 11: return -0.55557023301960222474;
        case 13: return -0.83146961230254523708;
        default: return -0.98078528040323044913;  // 15
    }
}
__host__ __device__ constexpr double sin32(int e) { return cos32(e - 8); }

// a * W_N^e with W_N = exp(-2 pi i / N) (forward) or exp(+2 pi i / N) (INV),
// N in {1, 2, 4, 8, 16, 32}; e is a compile-time constant after unrolling.
template <int N, bool INV, typename C>
__device__ __forceinline__ C mulw(C a, int e) {
    if constexpr (N == 32) {
        const int e32 = e & 31;
        if (!(e32 & 1)) return mulw<16, INV>(a, e32 / 2);
        using T = decltype(a.x);
        const T c = (T)cos32(e32);
        const T s = INV ? (T)sin32(e32) : (T)(-sin32(e32));
        return cmul(a, mk(c, s));
    }
    const int e16 = (e * (16 / N)) & 15;
    using T = decltype(a.x);
    if (e16 == 0) return a;
    if (e16 == 8) return mk(-a.x, -a.y);
    if (e16 == 4) return rot_quarter<INV>(a);
    if (e16 == 12) return rot_quarter<!INV>(a);
    const T c = (T)cos16(e16);
    const T s = INV ? (T)sin16(e16) : (T)(-sin16(e16));
    return cmul(a, mk(c, s));
}

// In-place DFT of N values v[0..N-1] (natural order in and out), N in
// {1,2,4,8,16,32}.  Two-factor decomposition N = A * B:
//   Y[n1][k2] = sum_{n2<B} v[n1 + A n2] W_B^{n2 k2}
//   Y[n1][k2] *= W_N^{n1 k2}
//   V[k2 + B k1] = sum_{n1<A} Y[n1][k2] W_A^{n1 k1}
template <int N, bool INV, typename C>
__device__ __forceinline__ void dft(C* v) {
    if constexpr (N == 1) {
        return;
    } else if constexpr (N == 2) {
        C a = v[0], b = v[1];
        v[0] = cadd(a, b);
        v[1] = csub(a, b);
    } else if constexpr (N == 4) {
        C s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
        C s13 = cadd(v[1], v[3]), d13 = rot_quarter<INV>(csub(v[1], v[3]));
        v[0] = cadd(s02, s13);
        v[2] = csub(s02, s13);
        v[1] = cadd(d02, d13);
        v[3] = csub(d02, d13);
    } else {
        constexpr int A = (N == 8) ? 2 : 4;
        constexpr int B = N / A;
        C y[A][B];
#pragma unroll
        for (int n1 = 0; n1 < A; ++n1) {
#pragma unroll
            for (int n2 = 0; n2 < B; ++n2) y[n1][n2] = v[n1 + A * n2];
            dft<B, INV>(y[n1]);
#pragma unroll
            for (int k2 = 0; k2 < B; ++k2) y[n1][k2] = mulw<N, INV>(y[n1][k2], n1 * k2);
        }
#pragma unroll
        for (int k2 = 0; k2 < B; ++k2) {
            C t[A];
#pragma unroll
            for (int n1 = 0; n1 < A; ++n1) t[n1] = y[n1][k2];
            dft<A, INV>(t);
#pragma unroll
            for (int k1 = 0; k1 < A; ++k1) v[k2 + B * k1] = t[k1];
        }
    }
}

// --------------------------------------------------------------------------
// Radix schedule of an R-point DFT done inside one CTA (R = 2^m <= 8192):
// sub-passes of the largest radix 2^ML (ML = 4: radix 16, the default; ML
// = 3: radix 8, for kernels that keep E = 8 values per thread), then one
// remainder radix last.
// --------------------------------------------------------------------------
__host__ __device__ constexpr int ilog2c(int n) { return n <= 1 ? 0 : 1 + ilog2c(n / 2); }
__host__ __device__ constexpr int n_steps(int R, int ML = 4) {
    return R <= (1 << ML) ? 1 : (ilog2c(R) / ML + ((ilog2c(R) % ML) ? 1 : 0));
}
__host__ __device__ constexpr int radix_at(int R, int s, int ML = 4) {
    return R <= (1 << ML) ? R : ((s < ilog2c(R) / ML) ? (1 << ML) : (1 << (ilog2c(R) % ML)));
}
__host__ __device__ constexpr int span_at(int R, int s, int ML = 4) {  // product of radices before step s
    return s == 0 ? 1 : span_at(R, s - 1, ML) * radix_at(R, s - 1, ML);
}

// offset of step s's twiddles in the step-major table of an R-point DFT:
// step s (s >= 1) owns (rho_s - 1) * Ns_s entries laid out [r - 1][k],
// value W_{Ns rho}^{k r}; consecutive k (consecutive threads) are adjacent.
__host__ __device__ constexpr int tw_off(int R, int s, int ML = 4) {
    return s <= 1 ? 0 : tw_off(R, s - 1, ML) + (radix_at(R, s - 1, ML) - 1) * span_at(R, s - 1, ML);
}
__host__ __device__ constexpr int tw_size(int R, int ML = 4) { return tw_off(R, n_steps(R, ML), ML); }
// all R = 2, 4, ..., 8192 tables concatenated (the ML = 4 set first, then
// the ML = 3 set, then the ML = 5 set of the radix-32 kernels): base offset
// of R's table
__host__ __device__ constexpr int tw_base_ml(int R, int ML) {
    return R <= 2 ? 0 : tw_base_ml(R / 2, ML) + tw_size(R / 2, ML);
}
__host__ __device__ constexpr int tw_base(int R, int ML = 4) {
    return ML == 4   ? tw_base_ml(R, 4)
           : ML == 3 ? tw_base_ml(16384, 4) + tw_base_ml(R, 3)
                     : tw_base_ml(16384, 4) + tw_base_ml(16384, 3) + tw_base_ml(R, 5);  // ML = 5
}
__host__ __device__ constexpr int tw_total() {
    return tw_base_ml(16384, 4) + tw_base_ml(16384, 3) + tw_base_ml(16384, 5);
}
// largest radix of a kernel holding E values per thread
__host__ __device__ constexpr int ml_of(int E) { return E >= 16 ? 4 : (E >= 8 ? 3 : 4); }

// padded shared-memory index: one spare slot every 16 elements (breaks the
// stride-16 bank pattern of the first Stockham write)
__device__ __forceinline__ int pad16(int i) { return i + (i >> 4); }
__host__ __device__ constexpr int pad16c(int i) { return i + (i >> 4); }

}  // namespace b200fft
