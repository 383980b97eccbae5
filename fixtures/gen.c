/*
 * fixtures/gen.c -- seeded synthetic inputs shared by the oracle side and the
 * CUDA side (the only code both sides use).  It holds none of the method's
 * arithmetic: no DFT, no twiddle, no filter -- only random numbers.
 *
 * Counter-based generator (reading R11): the value for global
 * element i of stream s under seed S is a pure function of (S, s, i), so the
 * same input comes out for any number of GPUs, threads or chunk offsets.
 *   key      = splitmix64(S * 0xD1B54A32D192ED03 ^ (s + 1) * 0x9E3779B97F4A7C15)
 *   word(c)  = splitmix64(key + (c + 1) * 0x9E3779B97F4A7C15)   (SplitMix64 output c)
 *   u(c)     = ((word(c) >> 11) + 0.5) * 2^-53          in (0, 1)
 * complex element i uses counters 2i (re) and 2i+1 (im):
 *   uniform[-1,1]: re = 2 u(2i) - 1, im = 2 u(2i+1) - 1
 *   normal(0,1)  : Box-Muller r = sqrt(-2 ln u(2i)), th = 2 pi u(2i+1),
 *                  re = r cos th, im = r sin th
 * computed in fp64; the float32 variants round once.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

static const double TWO_PI = 6.283185307179586476925286766559;

static inline uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static inline uint64_t stream_key(uint64_t seed, uint64_t stream) {
    return splitmix64(seed * 0xD1B54A32D192ED03ULL ^ (stream + 1) * 0x9E3779B97F4A7C15ULL);
}
static inline double u01(uint64_t key, uint64_t c) {
    uint64_t w = splitmix64(key + (c + 1) * 0x9E3779B97F4A7C15ULL);
    return ((double)(w >> 11) + 0.5) * (1.0 / 9007199254740992.0);
}

/* kind: 0 = uniform[-1,1], 1 = standard normal (Box-Muller) */
static inline void draw(uint64_t key, uint64_t i, int kind, double* re, double* im) {
    double a = u01(key, 2 * i), b = u01(key, 2 * i + 1);
    if (kind == 0) {
        *re = 2.0 * a - 1.0;
        *im = 2.0 * b - 1.0;
    } else {
        double r = sqrt(-2.0 * log(a)), th = TWO_PI * b;
        *re = r * cos(th);
        *im = r * sin(th);
    }
}

void fixtures_complex_f64(uint64_t seed, uint64_t stream, int kind, int64_t offset, int64_t count,
                          double* out) {
    const uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static) if (count >= 65536)
    for (int64_t i = 0; i < count; ++i)
        draw(key, (uint64_t)(offset + i), kind, out + 2 * i, out + 2 * i + 1);
}

void fixtures_complex_f32(uint64_t seed, uint64_t stream, int kind, int64_t offset, int64_t count,
                          float* out) {
    const uint64_t key = stream_key(seed, stream);
#pragma omp parallel for schedule(static) if (count >= 65536)
    for (int64_t i = 0; i < count; ++i) {
        double re, im;
        draw(key, (uint64_t)(offset + i), kind, &re, &im);
        out[2 * i] = (float)re;
        out[2 * i + 1] = (float)im;
    }
}

/*
 * Synthetic sky image (BASELINE configs[2]; reading R12), rows x cols
 * float32, row-major, pixel (row j, column i):
 *   background 100 + noise N(0, 5^2) per pixel (stream 0, re part of the
 *   Box-Muller pair of element j*cols+i)
 *   + nsrc point sources (stream 1, element s: x = cols*u(3s), y = rows*u(3s+1)
 *     continuous positions, flux F = 10^(2 + 3 u(3s+2)) log-uniform in
 *     [1e2, 1e5]) each blurred by a Gaussian PSF of sigma psf px:
 *     F / (2 pi psf^2) * exp(-((i-x)^2 + (j-y)^2) / (2 psf^2)),
 *     evaluated at integer pixel centres within 10 px, clipped at the edges.
 * Built in fp64, rounded once to float32.
 */
void fixtures_sky_image(uint64_t seed, int64_t rows, int64_t cols, int64_t nsrc, double psf,
                        float* out) {
    double* img = (double*)malloc(sizeof(double) * (size_t)(rows * cols));
    const uint64_t k0 = stream_key(seed, 0), k1 = stream_key(seed, 1);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < rows * cols; ++p) {
        double re, im;
        draw(k0, (uint64_t)p, 1, &re, &im);
        img[p] = 100.0 + 5.0 * re;
    }
    const int R = 10;
    for (int64_t s = 0; s < nsrc; ++s) {
        double x = (double)cols * u01(k1, 3 * (uint64_t)s);
        double y = (double)rows * u01(k1, 3 * (uint64_t)s + 1);
        double F = pow(10.0, 2.0 + 3.0 * u01(k1, 3 * (uint64_t)s + 2));
        double amp = F / (TWO_PI * psf * psf);
        int64_t ic = (int64_t)floor(x), jc = (int64_t)floor(y);
        for (int64_t j = jc - R; j <= jc + R; ++j) {
            if (j < 0 || j >= rows) continue;
            for (int64_t i = ic - R; i <= ic + R; ++i) {
                if (i < 0 || i >= cols) continue;
                double dx = (double)i - x, dy = (double)j - y;
                img[j * cols + i] += amp * exp(-(dx * dx + dy * dy) / (2.0 * psf * psf));
            }
        }
    }
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < rows * cols; ++p) out[p] = (float)img[p];
    free(img);
}
