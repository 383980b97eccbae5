/*
 * b200fft.h -- C ABI of the B200-native FFT library for the computation of
 * arXiv cs/0103001 (Higuera, Sarria, Fonseca, Idarraga, "Construction of an
 * algorithm in parallel for the Fast Fourier Transform").
 *
 * Citations "P:a-b" are line ranges of the paper's text, with the
 * section / equation they fall in.
 *
 * Operations (what is computed)
 * -----------------------------
 *  forward 1D  (Eq. E2 / Eq. coefFourier, Sec. 2):
 *      X[k] = (1/N) * sum_{j<N} x[j] * exp(-2 pi i j k / N)
 *  inverse 1D  (Eq. E3 at x_k = 2 pi k / N; Sec. 3):
 *      f[j] = sum_{k<N} c[k] * exp(+2 pi i j k / N)          (no 1/N)
 *  forward 2D  (eq5, Sec. 5), f is N x M row-major, N = rows:
 *      F(u,v) = (1/N) sum_x sum_y f(x,y) exp(-2 pi i (ux/N + vy/M))
 *  inverse 2D  (2D-IDFT):
 *      f(x,y) = (1/M) sum_u sum_v F(u,v) exp(+2 pi i (ux/N + vy/M))
 *  filter pipeline (Sec. 6): out = IDFT2( H .* DFT2(in) ), H real,
 *      multiplied into the real and imaginary parts.
 *
 * Conventions
 * -----------
 *  - Data are interleaved complex: complex64 = {float re, im} (8 B),
 *    complex128 = {double re, im} (16 B), batch-major, contiguous, in DEVICE
 *    memory owned by the caller (e.g. torch tensors).  Pointers must be
 *    aligned to the element size (8 / 16 B); otherwise FFT_E_INVALID_ARG.
 *  - Sizes are powers of two (the paper pads to the next power of two,
 *    P:366-367); anything else is FFT_E_INVALID_SIZE (see per-call limits).
 *  - Calls are asynchronous on the plan's stream (default: the legacy
 *    default stream; set it with fft_plan_set_stream).  Argument errors are
 *    returned synchronously; asynchronous CUDA faults surface on a later
 *    call.  After an error the output is undefined ("no partial result").
 *  - A plan is not thread-safe; distinct plans may be used concurrently.
 *  - CUDA graphs: a single-GPU call may be captured on the plan's stream
 *    after one warm-up call of the same kind (first calls allocate, set
 *    kernel attributes and upload tables), and replayed with new data in
 *    the captured buffers (per-launch state lives on the device).  Calls on
 *    distributed plans are not capturable: their barriers synchronise on the
 *    host or through the plan's NCCL communicator, and their receive slabs
 *    alternate between two phases on the host.
 *  - Nothing throws across this ABI; every call returns an fft_status, and
 *    fft_last_error() gives a thread-local detail string for the last
 *    failure.
 *  - There is no CPU fallback: every transform runs in the library's sm_100a
 *    kernels.
 */
#ifndef B200FFT_H
#define B200FFT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fft_plan_s* fft_plan; /* opaque, library-owned */

typedef enum {
    FFT_OK = 0,
    FFT_E_INVALID_SIZE = 1, /* n not a power of two, < 1, or over the limit */
    FFT_E_INVALID_ARG = 2,  /* null / misaligned pointer, bad rank, bad flag */
    FFT_E_UNSUPPORTED = 3,  /* valid request this build does not implement */
    FFT_E_CUDA = 4,         /* a CUDA runtime error (detail in fft_last_error) */
    FFT_E_NCCL = 5,         /* an NCCL error */
    FFT_E_ALLOC = 6,        /* device / host allocation failed */
    FFT_E_STATE = 7         /* call not valid in the plan's current state */
} fft_status;

typedef enum { FFT_C64 = 0, FFT_C128 = 1 } fft_precision;

typedef enum {
    FFT_FILTER_NONE = 0,  /* H = 1 */
    /* Gaussian low-pass of BASELINE configs[2]/[3]:
     *   H(u,v) = exp(-(k_u^2 / (2 s_N^2) + k_v^2 / (2 s_M^2))),
     *   k_u = u (u < N/2) else u - N (signed index), s_N = param * N / 2
     *   ("param * Nyquist"; param = 0.1 in the configs).  Square: the usual
     *   exp(-(kx^2+ky^2)/(2 (param Nyq)^2)). */
    FFT_FILTER_GAUSS = 1,
    /* Eq. (filtro), read literally on the unshifted spectrum:
     *   H = 0 if sqrt((u - N/2)^2 + (v - M/2)^2) <= b, else 1;  b = param. */
    FFT_FILTER_IDEAL_LITERAL = 2,
    /* The centred low-pass reading of Eq. (filtro):
     *   H = 1 if sqrt(k_u^2 + k_v^2) <= b, else 0 (signed k);  b = param. */
    FFT_FILTER_IDEAL_LOWPASS = 3
} fft_filter;

/* plan flags (fft_plan_create_ex) */
enum {
    FFT_FLAG_NONE = 0,
    /* fft2d_filter_pipeline input is float32 real [N][M] (promoted to complex
     * in the first pass's load, BASELINE configs[2]); output stays complex. */
    FFT_IN_REAL_F32 = 1u << 1,
    /* distributed single 1D transform (n = N1 N2, N1 = 2^ceil(m/2),
     * N2 = 2^floor(m/2)), fft_forward only: rank r keeps the four-step
     * transposed order -- X[k2 + N2 k1] for k2 in [r N2/P, (r+1) N2/P) at
     * local index (k2 - r N2/P) N1 + k1 -- one all-to-all less.  Ignored by
     * fft_inverse (its input is always in natural order). */
    FFT_OUT_TRANSPOSED = 1u << 0,
    /* NEXT-3 (with FFT_IN_REAL_F32, single GPU): fft2d_filter_pipeline
     * writes float32 real [N][M] -- the pipeline's real part.  For real
     * input and a real H with H(u, v) = H(-u, -v) (the Gaussian and both
     * readings of Eq. filtro) the pipeline preserves Hermitian symmetry, so
     * its imaginary part is zero in exact arithmetic (nothing is dropped).
     * The separable Gaussian on even sides 256..2048 runs as two real-to-real
     * row passes (two real rows per complex row); every other filter / size
     * (2 <= M, N, M <= 8192) goes through the half spectrum (the kernels of
     * fft_forward_r2c: R2C rows -> columns fwd * H * inv -> C2R rows). */
    FFT_OUT_REAL_F32 = 1u << 2
};

/* Short form from BASELINE.json's north_star: rank = transform
 * dimensionality (1: `batch` transforms of length n; 2: `batch` n x n grids),
 * complex64.  Limits: 1D n in [1, 2^30]; 2D n in [1, 8192] per side. */
fft_status fft_plan_create(fft_plan* out, int64_t n, int64_t batch, int rank);

/* dims[0..rank-1]: rank 1 -> {n}; rank 2 -> {N rows, M cols}.  flags: the
 * FFT_* flags above.  complex128 limits: 1D n <= 2^28, 2D sides <= 4096. */
fft_status fft_plan_create_ex(fft_plan* out, const int64_t* dims, int rank, int64_t batch,
                              fft_precision prec, unsigned flags);

/* cudaStream_t as void* (e.g. torch.cuda.current_stream().cuda_stream). */
fft_status fft_plan_set_stream(fft_plan plan, void* cuda_stream);

/* Scratch the plan needs for multi-pass transforms (0 if none).  If the
 * caller never calls fft_plan_set_workspace the library allocates it itself
 * on first use.  The caller keeps ownership of memory it passes in. */
size_t fft_plan_workspace_bytes(fft_plan plan);
fft_status fft_plan_set_workspace(fft_plan plan, void* dev_ptr, size_t bytes);

/* Note (complex64, n = 65536): the one-HBM-pass kernel keeps an
 * intermediate ring (~52 MiB, in the plan's workspace) in L2 through an
 * access-policy window and, on first use, sets the device's persisting-L2
 * set-aside (cudaLimitPersistingL2CacheSize) to the ring's size.  The
 * set-aside and the ring's persisting lines are released when the device's
 * last such plan is destroyed (cudaCtxResetPersistingL2Cache): until then
 * other kernels see that much less L2.  B200FFT_AB_PERSIST=0 leaves the
 * device limit alone (about 2.5% slower). */

/* Forward (1/N, or eq5's 1/N for rank 2) and inverse (unscaled, or the
 * 2D-IDFT's 1/M) transforms.  in/out: device pointers to the local data
 * (batch * prod(dims) elements); out may equal in. */
fft_status fft_forward(fft_plan plan, const void* in, void* out);
fft_status fft_inverse(fft_plan plan, const void* in, void* out);

/* Real data, Hermitian half spectrum (the paper's images are
 * real rasters).  A real signal's DFT satisfies X(-k) = conj
 * X(k), so bins 0 .. n/2 of each row determine it.
 *   fft_forward_r2c: rank 1: `batch` real rows of n -> n/2 + 1 bins each,
 *     X[k] = (1/n) sum_j x_j e^{-2 pi i jk/n} (Eq. E2), k = 0 .. n/2;
 *     rank 2: `batch` real N x M grids -> N x (M/2 + 1), eq5 (1/N)
 *     for columns v = 0 .. M/2.
 *   fft_inverse_c2r: rank 1: f_j = sum_{k<n} c_k e^{+2 pi i jk/n} (Eq. E3,
 *     unscaled) of the Hermitian spectrum with bins c_0 .. c_{n/2} (Im c_0
 *     and Im c_{n/2} are ignored, as a real signal has none); rank 2: the
 *     2D-IDFT (1/M) of the Hermitian grid given by its columns
 *     0 .. M/2.
 * Layouts (device, caller-owned, batch-major, contiguous): real rows of
 * float32 (FFT_C64 plans) or float64 (FFT_C128); half spectra of complex64 /
 * complex128 with row length n/2 + 1 (M/2 + 1).  The row length n (M) must
 * be >= 2 (FFT_E_INVALID_SIZE); in and out must not overlap
 * (FFT_E_INVALID_ARG if in == out); the 2D inverse uses the plan's workspace
 * and leaves `in` unchanged.  Not for distributed plans
 * (FFT_E_UNSUPPORTED).  Kernels: one R2C row kernel (a real row of n read as
 * the complex row of n/2 points x[2j] + i x[2j+1], one n/2-point transform,
 * the pairing of X[k] with X[n/2 - k] fused before its store) plus, for
 * rank 2, one column pass over the M/2 + 1 columns; C2R in reverse. */
fft_status fft_forward_r2c(fft_plan plan, const void* in_real, void* out_half);
fft_status fft_inverse_c2r(fft_plan plan, const void* in_half, void* out_real);

/* Rank-2 plans only: out = 2D-IDFT( H .* 2D-DFT(in) ) (Sec. 6).
 * The net scale of the round trip is 1/(N M) (eq5's 1/N times the
 * 2D-IDFT's 1/M), so H = 1 reproduces the input.  in is complex, or float32
 * real when the plan has FFT_IN_REAL_F32.  out may equal in only for
 * complex input. */
fft_status fft2d_filter_pipeline(fft_plan plan, const void* in, void* out, fft_filter filter,
                                 double param);

/* The paper's own application (Sec. 6), rank-2
 * complex64 single-GPU plans with N >= h, M >= w:
 *   in  : DEVICE uint8 [batch][h][w] row-major, a digital image with
 *         f(x,y) in Z+ u {0}; x = row.
 *   pad : zero-padded "on rows and on columns" to the plan's N x M
 *         (the usual N = next_pow2(h), M = next_pow2(w)), inside
 *         the first pass's load -- no padded copy.
 *   then: 2D DFT (eq5), spectrum, x H(u,v) into Re and Im,
 *         2D-IDFT: the fft2d_filter_pipeline computation with
 *         (filter, param); Eq. (filtro) with b = param for the ideal filters.
 *   out : DEVICE uint8 [batch][h][w]: real part of the filtered grid, rounded
 *         half up (floor(x + 0.5)), clamped to [0, max_val], cropped to the
 *         original h x w.  max_val in [1, 255].
 *   spectrum (optional, NULL to skip): DEVICE float32 [batch][N][M],
 *         |F(u,v)| = sqrt(Re^2 + Im^2) of the forward transform
 *         with eq5's 1/N, unshifted (u, v = 0 is the DC term).
 * Errors: FFT_E_INVALID_SIZE if h, w are outside [1, N] x [1, M];
 * FFT_E_INVALID_ARG for null pointers, a non-rank-2 / complex128 plan, a bad
 * filter or max_val; FFT_E_UNSUPPORTED on a distributed plan.  Uses the
 * plan's workspace (one complex N x M grid). */
fft_status fft2d_image_filter_u8(fft_plan plan, const uint8_t* in, int64_t h, int64_t w, uint8_t* out,
                                 fft_filter filter, double param, int max_val, float* spectrum);

/* NEXT-2: the paper's own parallel schedule (Sec. 4) for one
 * complex 1D transform of n = 2^m on P = 2^l ranks (a rank-1, batch-1 plan
 * with fft_plan_set_comm, or P virtual ranks on one GPU for tests):
 *   in : this rank's branch, the cyclic subsequence x[q + P j], j < n/P
 *        (the leaves processor idproc = q starts from); with
 *        virtual ranks, the P branches back to back (P x n/P elements).
 *   1. every rank transforms its branch (the tree's levels 1..m - l);
 *   2. l rounds (nproc_sup = P, P/2, ..., 2): ranks q in [S/2, S) send their
 *      vector to q - S/2 (NCCL send/recv over NVLink) and stop; the receiver
 *      combines the two with one radix-2 level;
 *   3. rank 0 (the MASTER) ends with X = (1/n) DFT(x) in natural order
 *      (P:191-224).
 *   out: rank 0: n elements (DEVICE, caller-owned); other ranks: unused (may
 *        be NULL).  Collective: every rank calls it.
 * It keeps the paper's serial tail (the last rounds run on half, then a
 * quarter ... of the GPUs, the last on rank 0 alone): a comparison point for
 * the all-to-all schedule of fft_forward, not its replacement.
 * Errors: FFT_E_INVALID_SIZE if P is not a power of two or does not divide
 * n; FFT_E_INVALID_ARG for a non-1D / batched plan or null pointers. */
fft_status fft_forward_paper_tree(fft_plan plan, const void* in, void* out);

/* End-to-end call on HOST buffers (pageable or pinned): copies the input
 * host->device, transforms, copies the result device->host, pipelined over
 * batch chunks (B200FFT_HOST_CHUNK_MB, default 64 MiB) on three plan-owned
 * streams: chunk c's copies overlap chunk c - 1's compute, while the computes
 * run one after another (they share the plan's workspace); returns after the
 * result is in host_out.  direction: +1 forward, -1 inverse, 0 filter
 * pipeline with (filter, param).  Ordered after the work already queued on
 * the plan's stream.  Same results as the device-pointer calls.
 * Errors: FFT_E_INVALID_ARG (null pointers, bad direction, pipeline on a
 * rank-1 plan), FFT_E_UNSUPPORTED (distributed or real-output plans),
 * FFT_E_ALLOC (the two device staging buffers per stream), FFT_E_CUDA. */
fft_status fft_execute_host(fft_plan plan, int direction, const void* host_in, void* host_out,
                            fft_filter filter, double param);

/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ----------------
 * Distributed plans shard the leading dimension across `nranks` processes:
 *  rank 1: the batch (independent transforms, no collective), or for
 *          batch == 1 the four-step view of one large transform (n/nranks
 *          contiguous elements per rank, all-to-all transposes);
 *  rank 2: row slabs of N/nranks rows per rank (all-to-all transposes).
 * Every rank calls every distributed entry point with identical plan
 * parameters (collective semantics, NCCL-style).
 * The all-to-alls are fused into the kernels by default: on the first
 * distributed call each rank allocates two receive slabs of its own (plan-
 * owned, 2 x the local slab; freed at destroy), maps every other rank's by
 * CUDA IPC (handles exchanged over the communicator; a collective decision,
 * so either all ranks use peer memory or none), and the row / transpose
 * kernels store into (and the final pass loads from) the other ranks' slabs
 * directly over NVLink, with stream-ordered NCCL barriers between the
 * phases (two per 2D grid; three per 1D four-step transform in natural
 * order, two with FFT_OUT_TRANSPOSED).  Asynchronous communicator errors
 * (ncclCommGetAsyncError) are polled after every distributed call and
 * returned as FFT_E_NCCL.
 * If any rank cannot map a peer, or B200FFT_P2P=0, the ncclSend/ncclRecv
 * all-to-all schedule runs instead (in the caller-visible workspace). */
fft_status fft_nccl_unique_id(unsigned char id[128]); /* on one rank; broadcast it */
/* Collective over the nranks processes: creates the plan's own NCCL
 * communicator (ncclCommInitRank).  After it, rank-2 plans take LOCAL slabs
 * (batch x N/nranks x M elements per call); rank-1 plans keep their own
 * (local) batch and run without any collective. */
fft_status fft_plan_set_comm(fft_plan plan, const unsigned char id[128], int nranks, int my_rank);
/* Tests on ONE GPU: the cross-process data plane of the fused schedules
 * without NCCL (NCCL refuses two ranks on one device).  The two collectives
 * of the fused schedules -- the IPC-handle all-gather (and the all-ranks-
 * mapped check) and the stream-ordered barrier -- are done by the caller's
 * host callbacks instead: allgather(ctx, mine, all, bytes) gathers `bytes`
 * from every rank into all[nranks * bytes] (rank order), barrier(ctx) blocks
 * until every rank has called it; both return 0 on success.  A barrier first
 * drains the plan's stream (cudaStreamSynchronize), so no kernel ever waits
 * on another process.  Everything else -- the slab layouts, the receive
 * slabs mapped by cudaIpcOpenMemHandle, the kernels' stores into and loads
 * from the other ranks' slabs, the schedule -- is the fft_plan_set_comm
 * path's.  Collective; same argument rules as fft_plan_set_comm; the
 * ncclSend/Recv all-to-all (B200FFT_P2P=0) and fft_forward_paper_tree are
 * NCCL-only (FFT_E_UNSUPPORTED).  The callbacks and ctx must stay valid
 * until fft_plan_destroy. */
typedef int (*fft_host_allgather_fn)(void* ctx, const void* mine, void* all, size_t bytes);
typedef int (*fft_host_barrier_fn)(void* ctx);
fft_status fft_plan_set_host_collectives(fft_plan plan, int nranks, int my_rank, fft_host_allgather_fn allgather,
                                        fft_host_barrier_fn barrier, void* ctx);
/* Tests / diagnostics: run the slab-decomposed schedule of a rank-2 plan (or
 * the four-step of a rank-1, batch-1 plan) as `nranks` virtual ranks on this
 * one GPU: the fused schedule with local slabs in place of peer memory
 * (B200FFT_DIST_EXCHANGE=1: the all-to-all schedule with device copies);
 * in/out stay the whole grid.  Same kernels and layouts as the NCCL path. */
fft_status fft_plan_set_virtual_ranks(fft_plan plan, int nranks);

fft_status fft_plan_destroy(fft_plan plan);

const char* fft_status_string(fft_status s);
const char* fft_last_error(void); /* thread-local detail of the last failure */

/* Introspection for tests/benchmarks: number of kernel launches the plan's
 * last call issued, and the library build string. */
int fft_plan_last_launch_count(fft_plan plan);
const char* fft_build_info(void);

/* Diagnostics: per-phase device timing.  With on != 0, each later call of
 * fft_forward / fft_inverse / fft2d_filter_pipeline records CUDA events on
 * the plan's stream between its phases -- for a distributed plan each
 * exchange (peer stores / loads or all-to-all), compute step and barrier
 * (the NVLink-exchange timing of the sharded configs, BASELINE north_star);
 * for a single-GPU call one phase.  fft_plan_phase_times waits for the last
 * call's final event, writes up to `max` phase durations in ms to `ms` and
 * their labels, ';'-separated and NUL-terminated, to `labels` (may be NULL),
 * and returns the number of phases (0 when profiling is off or no call ran).
 * Profiling adds one event record per phase; it is off by default. */
fft_status fft_plan_set_profiling(fft_plan plan, int on);
int fft_plan_phase_times(fft_plan plan, float* ms, int max, char* labels, size_t labels_bytes);

#ifdef __cplusplus
}
#endif
#endif /* B200FFT_H */
