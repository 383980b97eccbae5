/*
 * oracle/oracle.c -- the fp64 CPU oracle for the paper's DFT / FFT / 2D / filter
 * pipeline (arXiv cs/0103001, Higuera, Sarria, Fonseca, Idarraga).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this library.  The
 * product path (paper_cs_0103001_b200, libb200fft.so) never links, imports or
 * calls it, and shares no code, header, table or constant generator with it.
 *
 * Plain, slow, obviously-correct C in double precision.  No blocking, fusion or
 * reordering beyond what the paper's definitions/algorithms state.  Each
 * function cites the PAPER.md line range (P:a-b) and section/equation it
 * follows.  Complex arrays are interleaved (re, im) doubles.
 *
 * Pins (tests/test_oracle.py, -m "not gpu"): brute-force DFT (Eq. E2) for all
 * N <= 256, closed forms (impulse, constant, tone, [1,i,-1,-i]), Parseval,
 * linearity, numpy.fft (pocketfft) for N up to 2^20, the paper's bit-reversed
 * leaf order (tests/golden/tree_leaves_n8.txt), exp-polynomial interpolation
 * (Eq. E3), the Sec.3 reversal identity, the 2D brute-force double sum (eq5),
 * separable products, 2D Parseval, and the FFT-free spatial-convolution
 * closed form of the Gaussian pipeline.  Every function below is pinned; none
 * is "parity unpinned".
 *
 * Threading: the batched / 2D entry points use OpenMP over independent rows or
 * columns (or, for one huge transform, over butterflies inside a level).  The
 * arithmetic per element is identical to the single-threaded path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_E_SIZE 1
#define ORACLE_E_ARG 2
#define ORACLE_E_ALLOC 3

static const double TWO_PI = 6.283185307179586476925286766559;

static int is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }

static int ilog2(int64_t n) {
    int m = 0;
    while (((int64_t)1 << m) < n) ++m;
    return m;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_num_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}

/* ------------------------------------------------------------------------ */
/* Tree leaves: P:110-134 (Sec. 2), the level-0 row P_0 P_4 P_2 P_6 P_1 P_5  */
/* P_3 P_7 for N = 8.  Position p of the leaf row holds sample bitrev_m(p).   */
/* ------------------------------------------------------------------------ */
static int64_t bitrev(int64_t j, int m) {
    int64_t r = 0;
    for (int b = 0; b < m; ++b) {
        r = (r << 1) | (j & 1);
        j >>= 1;
    }
    return r;
}

int oracle_bitrev_order(int64_t n, int64_t* out) {
    if (!is_pow2(n)) return ORACLE_E_SIZE;
    if (!out) return ORACLE_E_ARG;
    int m = ilog2(n);
    for (int64_t p = 0; p < n; ++p) out[p] = bitrev(p, m);
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* The interpolation tree (Sec. 2), in place on C[0..N-1].        */
/*   level 0: the samples placed at the leaves in bit-reversed order;        */
/*   level n (n = 1..m): each node P^(n) of length L = 2^n combines its two   */
/*   children E = P^(n-1)_even, O = P^(n-1)_odd (each of length h = L/2):     */
/*        P[k]   = E[k] + w^k O[k]                                            */
/*        P[k+h] = E[k] - w^k O[k],      w^k = Z[k N / L] = e^{sign 2 pi i k/L}*/
/*   (the combine rule the paper leaves implicit).     */
/* Z_j = e^{-2 pi i j / N} is Table 2's twiddle vector; each      */
/* factor is computed directly from cos/sin of its own angle, never by        */
/* repeated multiplication.  sign = -1: forward sum; +1: the conjugate sum.   */
/* No normalisation here.                                                    */
/* ------------------------------------------------------------------------ */
static void tree_levels(double* C, int64_t N, int sign) {
    const int m = ilog2(N);
    /* level 0: bit-reversed leaves */
    for (int64_t j = 0; j < N; ++j) {
        int64_t r = bitrev(j, m);
        if (j < r) {
            double tr = C[2 * j], ti = C[2 * j + 1];
            C[2 * j] = C[2 * r];
            C[2 * j + 1] = C[2 * r + 1];
            C[2 * r] = tr;
            C[2 * r + 1] = ti;
        }
    }
    for (int n = 1; n <= m; ++n) {
        const int64_t L = (int64_t)1 << n, h = L >> 1;
        if (h <= 4096) {
            /* few distinct factors: compute each once, loop over the nodes */
            double* w = (double*)malloc(sizeof(double) * 2 * (size_t)h);
            for (int64_t k = 0; k < h; ++k) {
                double ang = sign * TWO_PI * (double)k / (double)L;
                w[2 * k] = cos(ang);
                w[2 * k + 1] = sin(ang);
            }
#pragma omp parallel for schedule(static) if (N >= 65536)
            for (int64_t s = 0; s < N; s += L) {
                for (int64_t k = 0; k < h; ++k) {
                    double* E = C + 2 * (s + k);
                    double* O = C + 2 * (s + k + h);
                    double tr = w[2 * k] * O[0] - w[2 * k + 1] * O[1];
                    double ti = w[2 * k] * O[1] + w[2 * k + 1] * O[0];
                    O[0] = E[0] - tr;
                    O[1] = E[1] - ti;
                    E[0] = E[0] + tr;
                    E[1] = E[1] + ti;
                }
            }
            free(w);
        } else {
            /* many factors, few nodes: one factor per k, loop over the nodes */
#pragma omp parallel for schedule(static)
            for (int64_t k = 0; k < h; ++k) {
                double ang = sign * TWO_PI * (double)k / (double)L;
                double wr = cos(ang), wi = sin(ang);
                for (int64_t s = 0; s < N; s += L) {
                    double* E = C + 2 * (s + k);
                    double* O = C + 2 * (s + k + h);
                    double tr = wr * O[0] - wi * O[1];
                    double ti = wr * O[1] + wi * O[0];
                    O[0] = E[0] - tr;
                    O[1] = E[1] - ti;
                    E[0] = E[0] + tr;
                    E[1] = E[1] + ti;
                }
            }
        }
    }
}

/* O2. Forward FFT = Eq. E2 / Eq. coefFourier:                     */
/*   H(k) = (1/N) sum_j f(x_j) e^{-2 pi i k j / N},                           */
/* evaluated by the tree above; the 1/N is applied once at the end.          */
int oracle_fft(const double* in, double* out, int64_t N) {
    if (!is_pow2(N)) return ORACLE_E_SIZE;
    if (!in || !out) return ORACLE_E_ARG;
    if (out != in) memcpy(out, in, sizeof(double) * 2 * (size_t)N);
    tree_levels(out, N, -1);
    const double s = 1.0 / (double)N;
#pragma omp parallel for schedule(static) if (N >= 65536)
    for (int64_t j = 0; j < 2 * N; ++j) out[j] *= s;
    return ORACLE_OK;
}

/* O3. Inverse FFT exactly as Sec. 3: evaluate the exponential    */
/* polynomial p (Eq. E3) with the forward FFT, multiply by N, and   */
/* read the result "in contrary order":                                      */
/*   f_k = p(x_k) = p(2 pi - x_{N-k}) = N * FFT(c)[(N - k) mod N].            */
/* Index 0 maps to itself (periodicity of p).  No 1/N on the inverse.        */
int oracle_ifft(const double* in, double* out, int64_t N) {
    if (!is_pow2(N)) return ORACLE_E_SIZE;
    if (!in || !out) return ORACLE_E_ARG;
    double* y = (double*)malloc(sizeof(double) * 2 * (size_t)N);
    if (!y) return ORACLE_E_ALLOC;
    oracle_fft(in, y, N);
    const double n = (double)N;
#pragma omp parallel for schedule(static) if (N >= 65536)
    for (int64_t k = 0; k < N; ++k) {
        int64_t src = (N - k) & (N - 1);
        out[2 * k] = n * y[2 * src];
        out[2 * k + 1] = n * y[2 * src + 1];
    }
    free(y);
    return ORACLE_OK;
}

/* Cross-check for O3: the same tree with the + sign and no scaling, i.e.    */
/* p(x_k) = sum_j c_j e^{+i j x_k}, x_k = 2 pi k / N (Eq. E3 at the nodes).    */
int oracle_ifft_plus_tree(const double* in, double* out, int64_t N) {
    if (!is_pow2(N)) return ORACLE_E_SIZE;
    if (!in || !out) return ORACLE_E_ARG;
    if (out != in) memcpy(out, in, sizeof(double) * 2 * (size_t)N);
    tree_levels(out, N, +1);
    return ORACLE_OK;
}

/* O9. Brute-force DFT: the plain double sum of Eq. E2 for any      */
/* N >= 1.  The integer product j*k is reduced mod N before it becomes an    */
/* angle.  inverse != 0: the unscaled + sign sum of Eq. E3 at x_k = 2pi k/N. */
int oracle_dft_bruteforce(const double* in, double* out, int64_t N, int inverse) {
    if (N < 1) return ORACLE_E_SIZE;
    if (!in || !out || in == out) return ORACLE_E_ARG;
    const double sign = inverse ? 1.0 : -1.0;
    const double scale = inverse ? 1.0 : 1.0 / (double)N;
#pragma omp parallel for schedule(static) if (N >= 1024)
    for (int64_t k = 0; k < N; ++k) {
        double sr = 0.0, si = 0.0;
        for (int64_t j = 0; j < N; ++j) {
            int64_t t = (int64_t)(((unsigned __int128)j * (unsigned __int128)k) % (unsigned __int128)N);
            double ang = sign * TWO_PI * (double)t / (double)N;
            double c = cos(ang), s = sin(ang);
            sr += in[2 * j] * c - in[2 * j + 1] * s;
            si += in[2 * j] * s + in[2 * j + 1] * c;
        }
        out[2 * k] = sr * scale;
        out[2 * k + 1] = si * scale;
    }
    return ORACLE_OK;
}

/* Eq. E3: p(x) = sum_k c_k e^{i k x}, direct summation.            */
int oracle_eval_exp_poly(const double* c, int64_t N, double x, double* out) {
    if (N < 1) return ORACLE_E_SIZE;
    if (!c || !out) return ORACLE_E_ARG;
    double sr = 0.0, si = 0.0;
    for (int64_t k = 0; k < N; ++k) {
        double ang = (double)k * x;
        double cr = cos(ang), s = sin(ang);
        sr += c[2 * k] * cr - c[2 * k + 1] * s;
        si += c[2 * k] * s + c[2 * k + 1] * cr;
    }
    out[0] = sr;
    out[1] = si;
    return ORACLE_OK;
}

/* Batched 1D: `batch` independent rows of length N, row-major.             */
int oracle_fft_batch(const double* in, double* out, int64_t N, int64_t batch, int inverse) {
    if (!is_pow2(N) || batch < 0) return ORACLE_E_SIZE;
    if ((!in || !out) && batch > 0) return ORACLE_E_ARG;
    int err = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : err)
    for (int64_t b = 0; b < batch; ++b) {
        const double* x = in + 2 * N * b;
        double* y = out + 2 * N * b;
        err |= inverse ? oracle_ifft(x, y, N) : oracle_fft(x, y, N);
    }
    return err ? ORACLE_E_ALLOC : ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* 2D (Sec. 5).  f is N x M, row-major: x = row index (0..N-1),   */
/* y = column index (0..M-1).                                                */
/* ------------------------------------------------------------------------ */
static void gather_col(const double* a, double* col, int64_t N, int64_t M, int64_t v) {
    for (int64_t x = 0; x < N; ++x) {
        col[2 * x] = a[2 * (x * M + v)];
        col[2 * x + 1] = a[2 * (x * M + v) + 1];
    }
}
static void scatter_col(double* a, const double* col, int64_t N, int64_t M, int64_t v) {
    for (int64_t x = 0; x < N; ++x) {
        a[2 * (x * M + v)] = col[2 * x];
        a[2 * (x * M + v) + 1] = col[2 * x + 1];
    }
}

/* O4 forward, eq5 by its factorisation:              */
/* "FFT on rows -> Multiplication for M -> FFT on columns":                  */
/*   F(x,v) = M * FFT_M(row x)[v]   (the unnormalised row sum),              */
/*   F(u,v) = FFT_N(column v of F(x,.))[u]   (carries eq5's 1/N).            */
int oracle_fft2d(const double* in, double* out, int64_t N, int64_t M) {
    if (!is_pow2(N) || !is_pow2(M)) return ORACLE_E_SIZE;
    if (!in || !out) return ORACLE_E_ARG;
    int err = 0;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : err)
    for (int64_t x = 0; x < N; ++x) {
        err |= oracle_fft(in + 2 * M * x, out + 2 * M * x, M);
        for (int64_t y = 0; y < 2 * M; ++y) out[2 * M * x + y] *= (double)M;
    }
#pragma omp parallel reduction(| : err)
    {
        double* col = (double*)malloc(sizeof(double) * 2 * (size_t)N);
        double* res = (double*)malloc(sizeof(double) * 2 * (size_t)N);
        if (!col || !res) err |= 1;
#pragma omp for schedule(dynamic, 4)
        for (int64_t v = 0; v < M; ++v) {
            if (!col || !res) continue;
            gather_col(out, col, N, M, v);
            oracle_fft(col, res, N);
            scatter_col(out, res, N, M, v);
        }
        free(col);
        free(res);
    }
    return err ? ORACLE_E_ALLOC : ORACLE_OK;
}

/* O4 inverse, the 2D-IDFT:                                      */
/*   f(x,y) = (1/M) sum_u sum_v F(u,v) e^{+i 2 pi (ux/N + vy/M)}             */
/* = (1/M) * [unscaled + sign sums over u (columns), then v (rows)], each    */
/* unscaled + sign 1D sum evaluated by the Sec. 3 inverse (oracle_ifft).     */
int oracle_ifft2d(const double* in, double* out, int64_t N, int64_t M) {
    if (!is_pow2(N) || !is_pow2(M)) return ORACLE_E_SIZE;
    if (!in || !out) return ORACLE_E_ARG;
    int err = 0;
    if (out != in) memcpy(out, in, sizeof(double) * 2 * (size_t)(N * M));
#pragma omp parallel reduction(| : err)
    {
        double* col = (double*)malloc(sizeof(double) * 2 * (size_t)N);
        double* res = (double*)malloc(sizeof(double) * 2 * (size_t)N);
        if (!col || !res) err |= 1;
#pragma omp for schedule(dynamic, 4)
        for (int64_t v = 0; v < M; ++v) {
            if (!col || !res) continue;
            gather_col(out, col, N, M, v);
            oracle_ifft(col, res, N);
            scatter_col(out, res, N, M, v);
        }
        free(col);
        free(res);
    }
    const double s = 1.0 / (double)M;
#pragma omp parallel for schedule(dynamic, 4) reduction(| : err)
    for (int64_t x = 0; x < N; ++x) {
        err |= oracle_ifft(out + 2 * M * x, out + 2 * M * x, M);
        for (int64_t y = 0; y < 2 * M; ++y) out[2 * M * x + y] *= s;
    }
    return err ? ORACLE_E_ALLOC : ORACLE_OK;
}

/* Brute-force 2D double sums, eq5 and the 2D-IDFT written out. */
int oracle_dft2d_bruteforce(const double* in, double* out, int64_t N, int64_t M, int inverse) {
    if (N < 1 || M < 1) return ORACLE_E_SIZE;
    if (!in || !out || in == out) return ORACLE_E_ARG;
    const double sign = inverse ? 1.0 : -1.0;
    const double scale = inverse ? 1.0 / (double)M : 1.0 / (double)N;
    for (int64_t u = 0; u < N; ++u)
        for (int64_t v = 0; v < M; ++v) {
            double sr = 0.0, si = 0.0;
            for (int64_t x = 0; x < N; ++x)
                for (int64_t y = 0; y < M; ++y) {
                    /* ux/N + vy/M as a fraction in [0,1) with exact integer reduction */
                    int64_t a = (u * x) % N, b = (v * y) % M;
                    double frac = (double)a / (double)N + (double)b / (double)M;
                    double ang = sign * TWO_PI * frac;
                    double c = cos(ang), s = sin(ang);
                    const double* f = in + 2 * (x * M + y);
                    sr += f[0] * c - f[1] * s;
                    si += f[0] * s + f[1] * c;
                }
            out[2 * (u * M + v)] = sr * scale;
            out[2 * (u * M + v) + 1] = si * scale;
        }
    return ORACLE_OK;
}

/* ------------------------------------------------------------------------ */
/* O5. Frequency filter H ("multiply it with the real and          */
/* imaginary part of the image's Fourier Transform").  The hot-path filter   */
/* is the Gaussian low-pass of BASELINE configs[2]/[3]:                       */
/*   H(u,v) = exp(-(k_u^2/(2 s_N^2) + k_v^2/(2 s_M^2))),                       */
/*   k_u = u for u < N/2 else u - N (signed DFT index), s_N = param * N/2     */
/*   (param = 0.1, "0.1 * Nyquist", Nyquist = N/2 in index units; DESIGN.md  */
/*   reading R7).  For square grids this is exp(-(k_u^2+k_v^2)/(2 s^2)).      */
/* Computed directly per (u,v) in fp64 -- not as a product of 1D tables.     */
/* ------------------------------------------------------------------------ */
int oracle_gauss_filter(int64_t N, int64_t M, double param, double* H) {
    if (N < 1 || M < 1) return ORACLE_E_SIZE;
    if (!H || !(param > 0.0)) return ORACLE_E_ARG;
    const double sN = param * (double)N / 2.0, sM = param * (double)M / 2.0;
#pragma omp parallel for schedule(static) if (N * M >= 65536)
    for (int64_t u = 0; u < N; ++u) {
        double ku = (double)(u < N / 2 ? u : u - N);
        if (N == 1) ku = 0.0;
        for (int64_t v = 0; v < M; ++v) {
            double kv = (double)(v < M / 2 ? v : v - M);
            if (M == 1) kv = 0.0;
            H[u * M + v] = exp(-(ku * ku / (2.0 * sN * sN) + kv * kv / (2.0 * sM * sM)));
        }
    }
    return ORACLE_OK;
}

/* O6. The image pipeline: 2D-FFT -> multiply Re and Im by H ->   */
/* 2D-IFFT.  H is any real N x M mask (row-major, fp64).                      */
int oracle_filter_pipeline(const double* in, double* out, int64_t N, int64_t M, const double* H) {
    if (!is_pow2(N) || !is_pow2(M)) return ORACLE_E_SIZE;
    if (!in || !out || !H) return ORACLE_E_ARG;
    double* F = (double*)malloc(sizeof(double) * 2 * (size_t)(N * M));
    if (!F) return ORACLE_E_ALLOC;
    int err = oracle_fft2d(in, F, N, M);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N * M; ++i) {
        F[2 * i] *= H[i];
        F[2 * i + 1] *= H[i];
    }
    err |= oracle_ifft2d(F, out, N, M);
    free(F);
    return err;
}

/* Convenience: O6 with the O5 Gaussian. */
int oracle_gauss_pipeline(const double* in, double* out, int64_t N, int64_t M, double param) {
    if (!is_pow2(N) || !is_pow2(M)) return ORACLE_E_SIZE;
    double* H = (double*)malloc(sizeof(double) * (size_t)(N * M));
    if (!H) return ORACLE_E_ALLOC;
    int err = oracle_gauss_filter(N, M, param, H);
    if (!err) err = oracle_filter_pipeline(in, out, N, M, H);
    free(H);
    return err;
}

/* ------------------------------------------------------------------------ */
/* O7. Sampled bins of one huge transform (N up to 2^30): the plain sum of   */
/* Eq. E2 for each requested k, with t = (j k) mod N exact in integers and    */
/* e^{-2 pi i t/N} = A[t >> h] * B[t & (2^h - 1)] (two fp64 tables of cos/sin */
/* computed directly).  Compensated (Kahan) summation inside blocks of 4096  */
/* terms, then pairwise over the block sums.  inverse: + sign, no 1/N.        */
/* ------------------------------------------------------------------------ */
static void kahan_add(double* s, double* c, double v) {
    double y = v - *c;
    double t = *s + y;
    *c = (t - *s) - y;
    *s = t;
}
static double pairwise(double* a, int64_t n) {
    if (n == 1) return a[0];
    if (n == 0) return 0.0;
    int64_t h = n / 2;
    return pairwise(a, h) + pairwise(a + h, n - h);
}
static int dft_bins_impl(const double* in, const float* in32, int64_t N, const int64_t* bins,
                         int64_t nbins, int inverse, double* out) {
    if (!is_pow2(N)) return ORACLE_E_SIZE;
    if ((!in && !in32) || !bins || !out) return ORACLE_E_ARG;
    const int m = ilog2(N);
    const int h = (m + 1) / 2;
    const int64_t nb = (int64_t)1 << h, na = (int64_t)1 << (m - h);
    const double sign = inverse ? 1.0 : -1.0;
    double* A = (double*)malloc(sizeof(double) * 2 * (size_t)na);
    double* B = (double*)malloc(sizeof(double) * 2 * (size_t)nb);
    const int64_t BLK = 4096;
    const int64_t nblk = (N + BLK - 1) / BLK;
    double* pr = (double*)malloc(sizeof(double) * (size_t)nblk);
    double* pi = (double*)malloc(sizeof(double) * (size_t)nblk);
    if (!A || !B || !pr || !pi) {
        free(A); free(B); free(pr); free(pi);
        return ORACLE_E_ALLOC;
    }
    for (int64_t i = 0; i < na; ++i) {
        double ang = sign * TWO_PI * (double)(i << h) / (double)N;
        A[2 * i] = cos(ang);
        A[2 * i + 1] = sin(ang);
    }
    for (int64_t i = 0; i < nb; ++i) {
        double ang = sign * TWO_PI * (double)i / (double)N;
        B[2 * i] = cos(ang);
        B[2 * i + 1] = sin(ang);
    }
    for (int64_t q = 0; q < nbins; ++q) {
        const uint64_t k = (uint64_t)bins[q] & (uint64_t)(N - 1);
#pragma omp parallel for schedule(static)
        for (int64_t blk = 0; blk < nblk; ++blk) {
            double sr = 0, cr = 0, si = 0, ci = 0;
            int64_t j1 = (blk + 1) * BLK < N ? (blk + 1) * BLK : N;
            for (int64_t j = blk * BLK; j < j1; ++j) {
                uint64_t t = ((uint64_t)j * k) & (uint64_t)(N - 1);
                const double* a = A + 2 * (t >> h);
                const double* b = B + 2 * (t & (uint64_t)(nb - 1));
                double wr = a[0] * b[0] - a[1] * b[1];
                double wi = a[0] * b[1] + a[1] * b[0];
                /* complex64 inputs are promoted exactly to fp64 (O1) */
                const double xr = in ? in[2 * j] : (double)in32[2 * j];
                const double xi = in ? in[2 * j + 1] : (double)in32[2 * j + 1];
                kahan_add(&sr, &cr, xr * wr - xi * wi);
                kahan_add(&si, &ci, xr * wi + xi * wr);
            }
            pr[blk] = sr;
            pi[blk] = si;
        }
        const double scale = inverse ? 1.0 : 1.0 / (double)N;
        out[2 * q] = pairwise(pr, nblk) * scale;
        out[2 * q + 1] = pairwise(pi, nblk) * scale;
    }
    free(A); free(B); free(pr); free(pi);
    return ORACLE_OK;
}

int oracle_dft_bins(const double* in, int64_t N, const int64_t* bins, int64_t nbins, int inverse,
                    double* out) {
    if (!in) return ORACLE_E_ARG;
    return dft_bins_impl(in, NULL, N, bins, nbins, inverse, out);
}

/* Same sums on a complex64 input (each value promoted exactly to fp64). */
int oracle_dft_bins_c64(const float* in, int64_t N, const int64_t* bins, int64_t nbins, int inverse,
                        double* out) {
    if (!in) return ORACLE_E_ARG;
    return dft_bins_impl(NULL, in, N, bins, nbins, inverse, out);
}
