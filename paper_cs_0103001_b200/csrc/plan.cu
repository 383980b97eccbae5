// plan.cu -- host side of libb200fft: plans, twiddle/filter tables, the
// C ABI of include/b200fft.h, and the execution schedules.
//
// Schedules:
//   1D, n <= 8192     : one launch of k_rows (whole transform per CTA line),
//                       1/N fused into the store (exact: a power of two).
//   1D, n > 8192      : 2 or 3 global Stockham passes (k_pass, radix
//                       128..1024), 1/N fused into the last pass.
//   2D (eq5)          : k_rows over the N rows (unnormalised: the paper's
//                       "FFT on rows -> multiplication for M"),
//                       then k_cols over the M columns with 1/N.
//   2D-IDFT           : k_cols inverse (unscaled), then k_rows inverse * 1/M.
//   filter pipeline   : k_rows fwd -> k_cols(fwd, * H/(N M), inv) -> k_rows inv
//                       (three launches; the column forward, the filter and
//                       the column inverse are one kernel).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#ifdef B200FFT_WITH_NCCL
#include <nccl.h>  // the torch wheel's NCCL 2.28 (not /usr/include's 2.27)
#endif

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: ranges for nsys / ncu --nvtx

#include "../../include/b200fft.h"
#include "fft_engine.cuh"
#include "launch.h"

using namespace b200fft;

#define B200FFT_STR2(x) #x
#define B200FFT_STR(x) B200FFT_STR2(x)

namespace {

thread_local std::string g_last_error;

// an NVTX range around each public entry point (a no-op without a tool)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

fft_status fail(fft_status s, const std::string& msg) {
    g_last_error = msg;
    return s;
}
fft_status cuda_fail(cudaError_t e, const char* what) {
    return fail(FFT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

bool is_pow2(int64_t n) { return n >= 1 && (n & (n - 1)) == 0; }
int ilog2(int64_t n) {
    int m = 0;
    while (((int64_t)1 << m) < n) ++m;
    return m;
}

// ---- twiddle tables -----------------------------------------------------
// All tables are computed in fp64 from cos/sin of the exactly reduced angle
// and rounded once to the plan's precision.
cudaError_t upload(const std::vector<double>& v, int prec, void** dptr) {
    size_t n = v.size();
    cudaError_t e;
    if (prec == 0) {
        std::vector<float> f(n);
        for (size_t i = 0; i < n; ++i) f[i] = (float)v[i];
        e = cudaMalloc(dptr, n * sizeof(float));
        if (e != cudaSuccess) return e;
        return cudaMemcpy(*dptr, f.data(), n * sizeof(float), cudaMemcpyHostToDevice);
    }
    e = cudaMalloc(dptr, n * sizeof(double));
    if (e != cudaSuccess) return e;
    return cudaMemcpy(*dptr, v.data(), n * sizeof(double), cudaMemcpyHostToDevice);
}

struct DeviceTables {
    void* tw[2] = {nullptr, nullptr};  // step-major in-CTA twiddles for c64 / c128
};

// The step-major twiddle tables of every in-CTA DFT size R = 2 .. 8192
// (fft_common.cuh tw_base / tw_off): entry [r - 1][k] of step s is
// W_{Ns rho}^{k r} = exp(-2 pi i k r / (Ns rho)).
void fill_step_tables(std::vector<double>& v) {
    static_assert(2 * RMAX == 16384, "tw_base's concatenation bound");
    const int total = tw_total();
    v.assign(2 * (size_t)total, 0.0);
    for (int ml = 5; ml >= 3; --ml)
    for (int R = 2; R <= RMAX; R *= 2) {
        for (int s = 1; s < n_steps(R, ml); ++s) {
            const int rho = radix_at(R, s, ml), Ns = span_at(R, s, ml);
            const int64_t n = (int64_t)Ns * rho;
            for (int r = 1; r < rho; ++r)
                for (int k = 0; k < Ns; ++k) {
                    const int64_t idx = (int64_t)tw_base(R, ml) + tw_off(R, s, ml) + (int64_t)(r - 1) * Ns + k;
                    const int64_t x = ((int64_t)k * r) % n;
                    const double ang = -2.0 * M_PI * (double)x / (double)n;
                    v[2 * idx] = std::cos(ang);
                    v[2 * idx + 1] = std::sin(ang);
                }
        }
    }
}
std::mutex g_tab_mu;
std::map<int, DeviceTables> g_tables;

cudaError_t device_twiddles(int dev, int prec, const void** out) {
    std::lock_guard<std::mutex> lk(g_tab_mu);
    DeviceTables& t = g_tables[dev];
    if (!t.tw[prec]) {
        std::vector<double> v;
        fill_step_tables(v);
        cudaError_t e = upload(v, prec, &t.tw[prec]);
        if (e != cudaSuccess) {
            t.tw[prec] = nullptr;
            return e;
        }
    }
    *out = t.tw[prec];
    return cudaSuccess;
}

}  // namespace

struct fft_plan_s {
    int rank = 1;
    int64_t n0 = 1, n1 = 1;  // 1D: n0 = length; 2D: n0 = N rows, n1 = M cols
    int64_t batch = 1;
    int prec = 0;
    unsigned flags = 0;
    int device = 0;
    cudaStream_t stream = nullptr;
    const void* tw = nullptr;
    // multi-pass 1D
    std::vector<int64_t> radices;
    std::vector<void*> pa, pb;  // per pass twiddle tables [r][k_lo], [r][k_hi]
    std::vector<int> klo_sh;
    // one-pass 65536-point 1D (fft_c2.cuh, n = cn1 * cn2): four-step twiddles [k2][n1]
    void* tw4 = nullptr;
    bool c2_acq = false;  // counted in the device's live 65536-point plans (kernels_c2.cu)
    // filter tables (Gaussian)
    void* gu = nullptr;
    void* gv = nullptr;
    double g_param = -1.0;
    // workspace
    void* ws = nullptr;
    size_t ws_bytes = 0;
    bool ws_owned = false;
    // host-execution staging buffers
    static constexpr int kHS = 3;          // host-execution streams (chunks round robin)
    void* hbuf[kHS] = {};                  // device output staging per stream
    void* hbin[kHS] = {};                  // device input staging per stream
    size_t hbuf_bytes = 0;
    cudaStream_t hstream[kHS] = {};
    cudaEvent_t hev = nullptr;
    cudaEvent_t hcomp[kHS] = {};  // end of a chunk's compute (fft_execute_host)
    int last_launches = 0;
    // distributed (slab decomposition of rank-2 plans)
    int nranks = 1, my_rank = 0;
    void* comm = nullptr;  // ncclComm_t owned by the plan
    // test mode (fft_plan_set_host_collectives): the IPC-handle all-gather and
    // the barriers are host callbacks instead of NCCL (comm stays null); the
    // data plane (IPC mappings, peer stores / loads by the kernels) is the same
    fft_host_allgather_fn hc_allgather = nullptr;
    fft_host_barrier_fn hc_barrier = nullptr;
    void* hc_ctx = nullptr;
    bool multi() const { return comm != nullptr || hc_barrier != nullptr; }
    int virt = 1;          // virtual ranks emulated on this GPU (tests), 1 = off
    // fused all-to-alls of the 2D slab schedule:
    // every rank's receive slabs (2 phases) mapped into every rank by CUDA IPC
    int p2p = 0;                       // 0 not decided, 1 on, -1 off (decided collectively)
    void* p2p_buf = nullptr;           // this rank's 2 receive slabs (owned)
    void* peer_buf[kMaxBlocks] = {};   // rank q's p2p_buf as mapped here
    void* bar_buf = nullptr;           // 1 float: the stream-ordered barrier
    void* ctl_buf = nullptr;           // 4 KiB for collective handshakes (allocated with the communicator)
    int64_t dist_phase = 0;            // receive slab of the next grid = phase & 1
    cudaEvent_t dev_ev = nullptr;
    // distributed four-step 1D (one transform of n = fs1 * fs2 over the ranks)
    int64_t fs1 = 0, fs2 = 0;
    fft_plan_s* sub_a = nullptr;  // length fs2, batch fs1 / P (step A)
    fft_plan_s* sub_b = nullptr;  // length fs1, batch fs2 / P (step B)
    void* fta = nullptr;          // W_n^{i << fsh}
    void* ftb = nullptr;          // W_n^{i}
    int fsh = 0;
    double scale_override = 0.0;  // sub-plans: scale of the last pass (0 = the default)
    // sub-plans: the outer four-step twiddle fused into the one-pass 32768-
    // point kernel (run_1d sets otw_done when it applied it)
    const void* otw_a = nullptr;
    const void* otw_b = nullptr;
    int otw_sh = 0;
    int64_t otw_row0 = 0;
    bool otw_done = false;
    // two-pass 2^30 (fft_big.cuh): W_32768^x, W_n^{i 32768}, W_n^i (i < 32768)
    void* big_twl = nullptr;
    void* big_hi = nullptr;
    void* big_lo = nullptr;
    // grid-barrier arrival count of the fused two-pass pipeline (k_rows_tma2;
    // plan-owned, zeroed once, only grows; each launch derives its target
    // from it on the device, so graph replays need no host-side state)
    unsigned long long* gbar = nullptr;
    // k_colfilt's task counters (plan-owned, grown on demand)
    void* cws = nullptr;
    size_t cws_bytes = 0;
    // real rows (NEXT-3): W_M^k, k < M/2 for the row length M (rtw_n = M)
    void* rtw = nullptr;
    int64_t rtw_n = 0;
    // four-step column passes of the Gaussian pipeline: W_N^x, x < N
    void* twl = nullptr;
    int64_t twl_n = 0;
    // the paper's own tree schedule (NEXT-2, fft_forward_paper_tree)
    fft_plan_s* tree_sub = nullptr;  // branch FFTs: length n / P, batch = local ranks
    void* tta = nullptr;             // W_n^{i << tsh}
    void* ttb = nullptr;             // W_n^{i}
    int tsh = 0;
    void* tws = nullptr;             // tree buffers (owned)
    size_t tws_bytes = 0;

    // per-phase device timing (fft_plan_set_profiling): event k marks the end
    // of phase k - 1 of the last call
    bool prof = false;
    std::vector<cudaEvent_t> pev;
    std::vector<std::string> plab;
    int pn = 0;

    size_t elem_bytes() const { return prec == 0 ? 8 : 16; }
    int P() const { return multi() ? nranks : virt; }
    // slab-decomposed schedule: a communicator (any size, 1 included) or virtual ranks
    bool dist() const { return (rank == 2 || batch == 1) && (multi() || virt > 1); }
    // elements addressed by one call: the local slab (NCCL) or everything (virtual)
    int64_t elems() const {
        if (rank == 1 && batch == 1 && multi()) return n0 / nranks;
        if (rank == 2 && multi()) return batch * (n0 / nranks) * n1;
        return batch * n0 * (rank == 2 ? n1 : 1);
    }
};

namespace {

// phase marks of the profiling mode (no-ops otherwise): prof_begin at the
// start of a call, prof_mark(label) after each phase, on the call's stream
void prof_mark(fft_plan_s* p, cudaStream_t st, const char* label) {
    if (!p->prof) return;
    if ((int)p->pev.size() <= p->pn) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) {
            p->prof = false;
            return;
        }
        p->pev.push_back(e);
        p->plab.emplace_back();
    }
    cudaEventRecord(p->pev[p->pn], st);
    if (p->pn > 0 && label) p->plab[p->pn - 1] = label;
    ++p->pn;
}
void prof_begin(fft_plan_s* p, cudaStream_t st) {
    if (!p->prof) return;
    p->pn = 0;
    prof_mark(p, st, nullptr);
}

size_t workspace_need(const fft_plan_s* p) {
    if (p->dist()) return 2 * (size_t)p->elems() * p->elem_bytes();  // send + recv slabs
    if (p->rank == 2)  // the transposed grid of the Gaussian pipeline (allocated on first use)
        return (size_t)p->n0 * p->n1 * p->elem_bytes();
    if (p->rank == 1 && p->tw4) return c2_workspace_bytes(p->batch, p->n0);
    if (p->rank == 1 && !p->radices.empty()) {
        size_t one = (size_t)p->elems() * p->elem_bytes();
        if (big_supported(p->prec, p->n0) && p->batch == 1 && !p->dist())
            return one + big_workspace_bytes();  // the two-pass 2^30: mid grid + L2 ring
        return p->radices.size() % 2 == 1 ? 2 * one : one;  // odd pass counts may need ws1 (run_1d)
    }
    return 0;
}

fft_status ensure_workspace(fft_plan_s* p) {
    size_t need = workspace_need(p);
    if (need == 0 || (p->ws && p->ws_bytes >= need)) return FFT_OK;
    if (p->ws && !p->ws_owned) return fail(FFT_E_STATE, "caller workspace smaller than fft_plan_workspace_bytes()");
    if (p->ws_owned && p->ws) cudaFree(p->ws);
    p->ws = nullptr;
    cudaError_t e = cudaMalloc(&p->ws, need);
    if (e != cudaSuccess) {
        p->ws = nullptr;
        return fail(FFT_E_ALLOC, std::string("workspace cudaMalloc: ") + cudaGetErrorString(e));
    }
    p->ws_bytes = need;
    p->ws_owned = true;
    return FFT_OK;
}

bool aligned(const void* ptr, size_t a) { return ((uintptr_t)ptr % a) == 0; }

// radix split of a multi-pass length L = 2^m (m >= 14): passes of radix
// <= 2^rmax, as even as possible (largest first).  rmax = 10 (2 or 3 passes
// of 128..1024) by default; complex64 transforms whose pass strides reach
// 2^21 elements (16 MiB) use rmax = 8 so that the pipelined pass kernel's
// tiles are 32 lines wide: 256-B runs instead of 64-B ones, which DRAM
// serves at 6.6 vs 2.9 TB/s at such strides (scripts/strided.cu,
// profiles/README.md) -- one pass more, each ~2x faster.
std::vector<int64_t> split_radices(int64_t L, int prec) {
    int m = ilog2(L);
    // complex64 from 2^21 on: radix <= 512, so every pass tile is 16 lines
    // wide (128-B runs: radix-1024 passes have 8-line tiles, 64-B runs, which
    // DRAM serves at half rate at multi-MiB strides) -- 2^30 in 4 passes at
    // ~5.9 TB/s each (11.6 ms) instead of 3 at 3.45 TB/s (14.9 ms)
    int rmax = (prec == 0 && m >= 21) ? 9 : 10;
    const char* rv = getenv("B200FFT_PASS_RMAX");
    if (rv) rmax = atoi(rv);
    int P = (m + rmax - 1) / rmax;
    std::vector<int64_t> r;
    for (int i = 0; i < P; ++i) {
        int mi = m / P + (i < m % P ? 1 : 0);
        r.push_back((int64_t)1 << mi);
    }
    // smaller radices first: the large-radix passes at the end stream a bit
    // faster (2^30: 128,128,256,256 25.5 ms fwd+inv vs 25.7 ms for
    // 256,256,128,128; 2^29: 128,128,128,256 best by ~1%)
    std::sort(r.begin(), r.end());
    // B200FFT_PASS_LOG2="7,8,8,7": an explicit pass order (log2 radices,
    // used when they sum to log2 L and each is 1..10)
    if (const char* ov = getenv("B200FFT_PASS_LOG2")) {
        std::vector<int64_t> o;
        int sum = 0;
        bool ok = true;
        for (const char* c = ov; *c;) {
            const int v = atoi(c);
            if (v < 1 || v > 10) ok = false;
            o.push_back((int64_t)1 << (v > 0 && v < 31 ? v : 1));
            sum += v;
            while (*c && *c != ',') ++c;
            if (*c == ',') ++c;
        }
        if (ok && sum == m) r = o;
    }
    return r;
}

fft_status run_1d(fft_plan_s* p, const void* in, void* out, bool inv, cudaStream_t st) {
    const int64_t L = p->n0;
    const double scale = p->scale_override != 0.0 ? p->scale_override : (inv ? 1.0 : 1.0 / (double)L);
    cudaError_t e;
    if (p->tw4) {
        // one HBM pass: the task pipeline reads each transform fully before
        // it writes it, so out == in is safe
        fft_status s = ensure_workspace(p);  // the Y ring and the task counters
        if (s != FFT_OK) return s;
        const bool fuse = p->otw_a && p->n0 == 32768;
        e = launch_c2(inv, p->n0, in, out, p->batch, scale, p->tw4, p->tw, p->ws, p->ws_bytes, st,
                      fuse ? p->otw_a : nullptr, p->otw_b, p->otw_sh, p->otw_row0);
        p->otw_done = fuse && e == cudaSuccess;
        p->last_launches = 1;
        if (e != cudaSuccess) return cuda_fail(e, "k_ab_ws launch");
        return FFT_OK;
    }
    if (big_supported(p->prec, L) && p->batch == 1 && !p->dist() && !p->radices.empty()) {
        // 2^30 in two HBM passes (fft_big.cuh): in -> ws (Y) -> out
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        if (!p->big_twl) {
            if (!p->c2_acq) {  // the ring's persisting set-aside is released with the plan
                c2_plan_acquire(p->device);
                p->c2_acq = true;
            }
            const int64_t Lh = 32768;
            std::vector<double> a(2 * Lh), hi(2 * Lh), lo(2 * Lh);
            for (int64_t x = 0; x < Lh; ++x) {
                const double t0 = -2.0 * M_PI * (double)x / (double)Lh;
                a[2 * x] = std::cos(t0);
                a[2 * x + 1] = std::sin(t0);
                const double t1 = -2.0 * M_PI * (double)(x * Lh) / (double)L;  // (x 2^15) / 2^30, exact
                hi[2 * x] = std::cos(t1);
                hi[2 * x + 1] = std::sin(t1);
                const double t2 = -2.0 * M_PI * (double)x / (double)L;
                lo[2 * x] = std::cos(t2);
                lo[2 * x + 1] = std::sin(t2);
            }
            e = upload(a, 0, &p->big_twl);
            if (e == cudaSuccess) e = upload(hi, 0, &p->big_hi);
            if (e == cudaSuccess) e = upload(lo, 0, &p->big_lo);
            if (e != cudaSuccess) return cuda_fail(e, "2^30 twiddle upload");
        }
        const size_t one = (size_t)L * p->elem_bytes();
        char* mid = (char*)p->ws;
        e = launch_big(inv, in, mid, out, scale, p->tw, p->big_twl, p->big_hi, p->big_lo, mid + one, p->ws_bytes - one,
                       st);
        p->last_launches = 2;
        if (e != cudaSuccess) return cuda_fail(e, "k_big launch");
        return FFT_OK;
    }
    if (p->radices.empty()) {
        e = launch_rows(p->prec, inv, false, L, in, out, p->batch, scale, p->tw, st);
        p->last_launches = 1;
        if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
        return FFT_OK;
    }
    fft_status s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    const int P = (int)p->radices.size();
    const size_t one = (size_t)p->elems() * p->elem_bytes();
    char* ws0 = (char*)p->ws;
    char* ws1 = ws0 + one;
    std::vector<const void*> src(P);
    std::vector<void*> dst(P);
    dst[P - 1] = out;
    // passes alternate between ws0 and out, ending in out; with an odd count
    // pass 0 would write out, which must not alias in (passes are not
    // in-place safe): then it writes ws1
    for (int i = 0; i < P - 1; ++i) dst[i] = ((P - 1 - i) % 2 == 0) ? out : (void*)ws0;
    if (P % 2 == 1 && in == out) dst[0] = ws1;
    src[0] = in;
    for (int i = 1; i < P; ++i) src[i] = dst[i - 1];
    int64_t Ns = 1;
    p->last_launches = 0;
    for (int i = 0; i < P; ++i) {
        const int64_t R = p->radices[i];
        e = launch_pass(p->prec, inv, R, src[i], dst[i], L, Ns, p->batch, (i == P - 1) ? scale : 1.0, p->tw,
                        p->pa[i], p->pb[i], p->klo_sh[i], st);
        p->last_launches++;
        if (e != cudaSuccess) return cuda_fail(e, "k_pass launch");
        Ns *= R;
    }
    return FFT_OK;
}

fft_status run_2d(fft_plan_s* p, const void* in, void* out, bool inv, cudaStream_t st) {
    const int64_t N = p->n0, M = p->n1;
    FilterArgs f{};
    cudaError_t e;
    if (!inv) {
        // rows: unnormalised (FFT_M * M)
        e = launch_rows(p->prec, false, false, M, in, out, p->batch * N, 1.0, p->tw, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
        // columns: eq5's 1/N
        e = launch_cols(p->prec, 0, N, out, out, M, p->batch, 1.0 / (double)N, p->tw, f, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_cols launch");
    } else {
        e = launch_cols(p->prec, 1, N, in, out, M, p->batch, 1.0, p->tw, f, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_cols launch");
        e = launch_rows(p->prec, true, false, M, out, out, p->batch * N, 1.0 / (double)M, p->tw, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
    }
    p->last_launches = 2;
    return FFT_OK;
}

fft_status gauss_tables(fft_plan_s* p, double param) {
    if (p->gu && p->g_param == param) return FFT_OK;
    if (p->gu) cudaFree(p->gu);
    if (p->gv) cudaFree(p->gv);
    p->gu = p->gv = nullptr;
    auto make = [&](int64_t n, void** d) -> cudaError_t {
        std::vector<double> g(n);
        const double s = param * (double)n / 2.0;
        for (int64_t u = 0; u < n; ++u) {
            const double k = (double)(u < n / 2 ? u : u - n);
            g[u] = (n == 1) ? 1.0 : std::exp(-k * k / (2.0 * s * s));
        }
        if (p->prec == 0) {
            std::vector<float> f(g.begin(), g.end());
            cudaError_t e = cudaMalloc(d, n * sizeof(float));
            if (e != cudaSuccess) return e;
            return cudaMemcpy(*d, f.data(), n * sizeof(float), cudaMemcpyHostToDevice);
        }
        cudaError_t e = cudaMalloc(d, n * sizeof(double));
        if (e != cudaSuccess) return e;
        return cudaMemcpy(*d, g.data(), n * sizeof(double), cudaMemcpyHostToDevice);
    };
    cudaError_t e = make(p->n0, &p->gu);
    if (e == cudaSuccess) e = make(p->n1, &p->gv);
    if (e != cudaSuccess) return cuda_fail(e, "filter table upload");
    p->g_param = param;
    return FFT_OK;
}

// programmatic dependent launch of a pipeline's second row pass
// (B200FFT_PDL=0 turns it off)
bool pdl_on() { return pdl_enabled(); }

// W_N^x, x < N (fp64-generated): the twiddles of the four-step column passes
cudaError_t ensure_twl(fft_plan_s* p, int64_t N) {
    if (p->twl_n == N) return cudaSuccess;
    if (p->twl) cudaFree(p->twl);
    p->twl = nullptr;
    p->twl_n = 0;
    std::vector<double> t(2 * (size_t)N);
    for (int64_t x = 0; x < N; ++x) {
        const double ang = -2.0 * M_PI * (double)x / (double)N;
        t[2 * x] = std::cos(ang);
        t[2 * x + 1] = std::sin(ang);
    }
    cudaError_t e = upload(t, p->prec, &p->twl);
    if (e == cudaSuccess) p->twl_n = N;
    return e;
}

// W_M^k, k < M/2 (fp64-generated, rounded once): the R2C / C2R pairing twiddles
cudaError_t ensure_rtw(fft_plan_s* p, int64_t M) {
    if (p->rtw_n == M) return cudaSuccess;
    if (p->rtw) cudaFree(p->rtw);
    if (p->cws) cudaFree(p->cws);
    if (p->big_twl) cudaFree(p->big_twl);
    if (p->big_hi) cudaFree(p->big_hi);
    if (p->big_lo) cudaFree(p->big_lo);
    p->rtw = nullptr;
    p->rtw_n = 0;
    const int64_t h = M / 2 > 0 ? M / 2 : 1;
    std::vector<double> t(2 * (size_t)h);
    for (int64_t k = 0; k < h; ++k) {
        const double ang = -2.0 * M_PI * (double)k / (double)M;
        t[2 * k] = std::cos(ang);
        t[2 * k + 1] = std::sin(ang);
    }
    cudaError_t e = upload(t, p->prec, &p->rtw);
    if (e == cudaSuccess) p->rtw_n = M;
    return e;
}

// NEXT-3: real input -> Hermitian half spectrum.  rank 1: Eq. E2 (1/n) of
// each row, bins 0 .. n/2; rank 2: eq5 (rows unnormalised, columns 1/N) on
// columns v = 0 .. M/2.
fft_status run_r2c(fft_plan_s* p, const void* in, void* out, cudaStream_t st) {
    const int64_t N = p->n0, M = p->rank == 2 ? p->n1 : p->n0;
    cudaError_t e = ensure_rtw(p, M);
    if (e != cudaSuccess) return cuda_fail(e, "R2C twiddle upload");
    const int64_t rows = p->rank == 2 ? p->batch * N : p->batch;
    e = launch_rows_r2c(p->prec, M, in, out, rows, p->rank == 2 ? 1.0 : 1.0 / (double)M, p->tw, p->rtw, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_rows_r2c launch");
    p->last_launches = 1;
    if (p->rank == 2) {
        FilterArgs f{};
        e = launch_cols(p->prec, 0, N, out, out, M / 2 + 1, p->batch, 1.0 / (double)N, p->tw, f, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_cols launch");
        p->last_launches = 2;
    }
    return FFT_OK;
}

// NEXT-3: Hermitian half spectrum -> real.  rank 1: Eq. E3 (unscaled);
// rank 2: 2D-IDFT (columns unscaled, rows 1/M).  `in` is not modified for
// rank 1; rank 2 uses the workspace for the column pass.
fft_status run_c2r(fft_plan_s* p, const void* in, void* out, cudaStream_t st) {
    const int64_t N = p->n0, M = p->rank == 2 ? p->n1 : p->n0;
    cudaError_t e = ensure_rtw(p, M);
    if (e != cudaSuccess) return cuda_fail(e, "C2R twiddle upload");
    if (p->rank == 1) {
        e = launch_rows_c2r(p->prec, M, in, out, p->batch, 1.0, p->tw, p->rtw, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_rows_c2r launch");
        p->last_launches = 1;
        return FFT_OK;
    }
    fft_status s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    const size_t half = (size_t)N * (M / 2 + 1) * p->elem_bytes();
    for (int64_t g = 0; g < p->batch; ++g) {
        FilterArgs f{};
        e = launch_cols(p->prec, 1, N, (const char*)in + g * half, p->ws, M / 2 + 1, 1, 1.0, p->tw, f, st);
        if (e == cudaSuccess)
            e = launch_rows_c2r(p->prec, M, p->ws, (char*)out + g * (size_t)N * M * (p->prec == 0 ? 4 : 8), N,
                                1.0 / (double)M, p->tw, p->rtw, st);
        if (e != cudaSuccess) return cuda_fail(e, "C2R launch");
    }
    p->last_launches = (int)(2 * p->batch);
    return FFT_OK;
}

// NEXT-3: real in, real out through the half spectrum for ANY filter whose H
// is real with H(u, v) = H(-u, -v) (the Gaussian and both readings of Eq.
// filtro): R2C rows -> columns fwd (1/N) x H x inv -> C2R rows (1/M); half
// the bytes and flops of the complex pipeline.
cudaError_t colfilt(fft_plan_s* p, void* grid, int64_t SM, int64_t nimg, double scale, const void* gv,
                    int64_t col_off, cudaStream_t st);

fft_status run_pipeline_half(fft_plan_s* p, const void* in, void* out, const FilterArgs& f, cudaStream_t st) {
    const int64_t N = p->n0, M = p->n1;
    cudaError_t e = ensure_rtw(p, M);
    if (e != cudaSuccess) return cuda_fail(e, "R2C twiddle upload");
    fft_status s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    const size_t grid_r = (size_t)N * M * sizeof(float);
    // the Gaussian on 8192 rows: the half spectrum with rows padded to
    // M/2 + 16 bins (a multiple of 16; the pad bins are never read back) so
    // the one-pass column filter k_colfilt takes all its columns, applying
    // g_N(u) g_M(v) / (N M) (its g_M-per-column mode); 0.50 -> ~0.25 ms for
    // the 8192^2 column pass against k_cols' 8192-long column tiles
    if (f.kind == FFT_FILTER_GAUSS && p->prec == 0 && N == 8192 && M >= 32 && colfilt_supported(N, M)) {
        const int64_t ld = M / 2 + 16;
        for (int64_t g = 0; g < p->batch; ++g) {
            e = launch_rows_r2c(p->prec, M, (const char*)in + g * grid_r, p->ws, N, 1.0, p->tw, p->rtw, st, ld);
            if (e == cudaSuccess) e = colfilt(p, p->ws, ld, 1, 1.0 / ((double)N * (double)M), p->gv, 0, st);
            if (e == cudaSuccess)
                e = launch_rows_c2r(p->prec, M, p->ws, (char*)out + g * grid_r, N, 1.0, p->tw, p->rtw, st, ld);
            if (e != cudaSuccess) return cuda_fail(e, "half-spectrum pipeline (k_colfilt) launch");
        }
        p->last_launches = (int)(3 * p->batch);
        return FFT_OK;
    }
    for (int64_t g = 0; g < p->batch; ++g) {
        e = launch_rows_r2c(p->prec, M, (const char*)in + g * grid_r, p->ws, N, 1.0, p->tw, p->rtw, st);
        if (e == cudaSuccess)
            e = launch_cols(p->prec, 2, N, p->ws, p->ws, M / 2 + 1, 1, 1.0 / ((double)N * (double)M), p->tw, f, st);
        if (e == cudaSuccess)
            e = launch_rows_c2r(p->prec, M, p->ws, (char*)out + g * grid_r, N, 1.0, p->tw, p->rtw, st);
        if (e != cudaSuccess) return cuda_fail(e, "half-spectrum pipeline launch");
    }
    p->last_launches = (int)(3 * p->batch);
    return FFT_OK;
}

// the one-pass column filter (k_colfilt) on [nimg][8192][SM] with its own
// counter buffer; scale and g_M (gv, with the slab's column offset) as the
// caller's schedule needs
cudaError_t colfilt(fft_plan_s* p, void* grid, int64_t SM, int64_t nimg, double scale, const void* gv,
                    int64_t col_off, cudaStream_t st) {
    cudaError_t e = ensure_twl(p, p->n0);
    if (e != cudaSuccess) return e;
    const size_t need = colfilt_workspace_bytes(SM, nimg);
    if (p->cws_bytes < need) {
        if (p->cws) cudaFree(p->cws);
        p->cws = nullptr;
        p->cws_bytes = 0;
        e = cudaMalloc(&p->cws, need);
        if (e != cudaSuccess) return e;
        p->cws_bytes = need;
    }
    return launch_colfilt(grid, SM, nimg, scale, p->tw, p->twl, p->gu, gv, col_off, p->cws, p->cws_bytes, st);
}

// the fused pipeline's grid-barrier count (zeroed once; only grows)
cudaError_t ensure_gbar(fft_plan_s* p, cudaStream_t st) {
    if (p->gbar) return cudaSuccess;
    cudaError_t e = cudaMalloc(&p->gbar, 256);
    if (e == cudaSuccess) e = cudaMemsetAsync(p->gbar, 0, 256, st);
    return e;
}

fft_status run_pipeline(fft_plan_s* p, const void* in, void* out, fft_filter filter, double param,
                        cudaStream_t st) {
    const int64_t N = p->n0, M = p->n1;
    FilterArgs f{};
    f.kind = (int)filter;
    f.N = N;
    f.M = M;
    if (filter == FFT_FILTER_GAUSS) {
        fft_status s = gauss_tables(p, param);
        if (s != FFT_OK) return s;
        f.gu = p->gu;
        f.gv = p->gv;
    } else if (filter == FFT_FILTER_IDEAL_LITERAL || filter == FFT_FILTER_IDEAL_LOWPASS) {
        f.b2 = param * param;
    }
    const bool real_in = (p->flags & FFT_IN_REAL_F32) != 0;
    cudaError_t e;
    // Separable filter (the Gaussian, H = g_N(u) g_M(v)): the row and column
    // operators commute, so IDFT2(H DFT2 f) = [IDFT_c g_N DFT_c][IDFT_r g_M
    // DFT_r] f exactly -- two fused passes (rows fwd*g*inv, then columns
    // fwd*g*inv), 32 B/point of HBM instead of 48 (DESIGN.md "Separable
    // pipeline").  B200FFT_PIPE_LITERAL=1 keeps the three-pass order.
    if (p->flags & FFT_OUT_REAL_F32) {
        // NEXT-3: real in, real out.  The separable Gaussian on sides
        // 256..2048 takes two real rows per complex line in both passes (the
        // Gaussian row / column operators are real and even: two launches);
        // every other filter and size goes through the half spectrum.
        const char* hs = getenv("B200FFT_PIPE_HALF");
        if (!real_in || M < 2) return fail(FFT_E_UNSUPPORTED, "real-output pipeline needs real input and M >= 2");
        if (filter != FFT_FILTER_GAUSS || N % 2 || M % 2 || !rows_filter_transposed_supported(p->prec, M) ||
            !rows_filter_transposed_supported(p->prec, N) || (hs && hs[0] == '1'))
            return run_pipeline_half(p, in, out, f, st);
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        const size_t grid = (size_t)N * M * sizeof(float);
        for (int64_t g = 0; g < p->batch; ++g) {
            e = launch_rows_filter_transposed(false, M, (const char*)in + g * grid, p->ws, N / 2, 1.0 / (double)M, p->tw,
                                              p->gv, st, true);
            if (e == cudaSuccess)
                e = launch_rows_filter_transposed(false, N, p->ws, (char*)out + g * grid, M / 2, 1.0 / (double)N,
                                                  p->tw, p->gu, st, 1, pdl_on());
            if (e != cudaSuccess) return cuda_fail(e, "k_rows_tma (real pairs) launch");
        }
        p->last_launches = (int)(2 * p->batch);
        return FFT_OK;
    }
    const char* lit_env = getenv("B200FFT_PIPE_LITERAL");
    const bool literal = lit_env && lit_env[0] == '1';
    const char* rp_env = getenv("B200FFT_PIPE_REALPAIR");
    if (real_in && filter == FFT_FILTER_GAUSS && !literal && !(rp_env && rp_env[0] == '0') && N % 2 == 0 &&
        M % 2 == 0 && rows_filter_transposed_supported(p->prec, M) && rows_filter_transposed_supported(p->prec, N)) {
        // real input, Gaussian (real, even, separable): the pipeline's exact
        // output is real (R20), so both passes take two real rows
        // per complex line (NEXT-3's pairs) and the second stores the complex
        // grid with imaginary parts 0 -- half the arithmetic and 80 MiB of
        // HBM traffic instead of 112 MiB for C3
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        const size_t in_grid = (size_t)N * M * sizeof(float);
        const size_t grid = (size_t)N * M * p->elem_bytes();
        // square grids: both passes in one cooperative launch (C3: 38.9 vs
        // 39.9 us; the real-output form measured 1 us slower fused, so it
        // keeps the two launches with PDL)
        if (rows_filter2_supported(p->prec, N, M)) {
            if ((e = ensure_gbar(p, st)) != cudaSuccess) return cuda_fail(e, "grid barrier counter");
            for (int64_t g = 0; g < p->batch; ++g) {
                e = launch_rows_filter2(M, (const char*)in + g * in_grid, p->ws, (char*)out + g * grid,
                                        1.0 / (double)M, p->gv, 1.0 / (double)N, p->gu, p->tw, 2, p->gbar, st);
                if (e != cudaSuccess) return cuda_fail(e, "k_rows_tma2 (real pairs, complex out) launch");
            }
            p->last_launches = (int)p->batch;
            return FFT_OK;
        }
        for (int64_t g = 0; g < p->batch; ++g) {
            e = launch_rows_filter_transposed(false, M, (const char*)in + g * in_grid, p->ws, N / 2, 1.0 / (double)M,
                                              p->tw, p->gv, st, 1);
            if (e == cudaSuccess)
                e = launch_rows_filter_transposed(false, N, p->ws, (char*)out + g * grid, M / 2, 1.0 / (double)N,
                                                  p->tw, p->gu, st, 2, pdl_on());
            if (e != cudaSuccess) return cuda_fail(e, "k_rows_tma (real pairs, complex out) launch");
        }
        p->last_launches = (int)(2 * p->batch);
        return FFT_OK;
    }
    if (filter == FFT_FILTER_GAUSS && !literal && rows_filter_transposed_supported(p->prec, M) &&
        rows_filter_transposed_supported(p->prec, N)) {
        // both passes as contiguous-row kernels with transposed stores:
        // in [N][M] -> (rows: fwd * g_M / M * inv) -> ws [M][N] -> (rows:
        // fwd * g_N / N * inv) -> out [N][M]
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        const size_t in_grid = (size_t)N * M * (real_in ? 4 : p->elem_bytes());
        const size_t grid = (size_t)N * M * p->elem_bytes();
        for (int64_t g = 0; g < p->batch; ++g) {
            e = launch_rows_filter_transposed(real_in, M, (const char*)in + g * in_grid, p->ws, N, 1.0 / (double)M,
                                              p->tw, p->gv, st);
            if (e == cudaSuccess)
                e = launch_rows_filter_transposed(false, N, p->ws, (char*)out + g * grid, M, 1.0 / (double)N, p->tw,
                                                  p->gu, st, 0, pdl_on());
            if (e != cudaSuccess) return cuda_fail(e, "k_rows_tma (transposed) launch");
        }
        p->last_launches = (int)(2 * p->batch);
        return FFT_OK;
    }
    // rows pass (fwd * g_M * inv) -> the column direction as a four-step
    // over N = 64 N2: A = column DFT over the
    // 64 rows N2 apart + twiddle W_N^{n2 k1}; B = fwd * g_N[k1 + 64 k2] / N *
    // inv over each block of N2 consecutive rows; A' = conj twiddle + inverse
    // over the 64 rows.  No transposes, no 8192-long column lines.
    const char* c4_env = getenv("B200FFT_PIPE_COLS4");
    const bool c4_default = true;  // 1060 us vs 1130 us for the transposes path (C4, profiles/README.md)
    if (filter == FFT_FILTER_GAUSS && !literal && p->prec == 0 && N >= 4096 && N <= 8192 && M >= 256 &&
        M <= 8192 && (c4_env ? c4_env[0] == '1' : c4_default)) {
        e = ensure_twl(p, N);
        if (e != cudaSuccess) return cuda_fail(e, "column twiddle upload");
        const int64_t N1 = 64, N2 = N / 64;
        const size_t in_grid = (size_t)N * M * (real_in ? 4 : p->elem_bytes());
        const size_t grid = (size_t)N * M * p->elem_bytes();
        FilterArgs fa{};
        fa.tw_l = p->twl;
        fa.tdiv = M;
        FilterArgs fb{};
        fb.kind = 6;
        fb.gu = p->gu;
        fb.n1 = N1;
        if (colfilt_supported(N, M)) {
            // the three column phases as ONE task-pipeline kernel, each group
            // of 16 columns staying in L2 between them (fft_colpipe.cuh):
            // rows pass + 1 column pass = one HBM read + write per pass
            e = launch_rows(p->prec, false, real_in, M, in, out, p->batch * N, 1.0 / (double)M, p->tw, st, -1, -1,
                            p->gv);
            if (e == cudaSuccess) e = colfilt(p, out, M, p->batch, 1.0 / (double)N, nullptr, 0, st);
            if (e != cudaSuccess) return cuda_fail(e, "one-pass column pipeline launch");
            p->last_launches = 2;
            return FFT_OK;
        }
        for (int64_t g = 0; g < p->batch; ++g) {
            char* o = (char*)out + g * grid;
            e = launch_rows(p->prec, false, real_in, M, (const char*)in + g * in_grid, o, N, 1.0 / (double)M, p->tw,
                            st, -1, -1, p->gv);
            if (e == cudaSuccess) e = launch_cols_fourstep(3, N1, o, o, N2 * M, 1, 1.0, p->tw, fa, st);
            if (e == cudaSuccess) e = launch_cols_fourstep(2, N2, o, o, M, N1, 1.0 / (double)N, p->tw, fb, st);
            if (e == cudaSuccess) e = launch_cols_fourstep(4, N1, o, o, N2 * M, 1, 1.0, p->tw, fa, st);
            if (e != cudaSuccess) return cuda_fail(e, "four-step column pipeline launch");
        }
        p->last_launches = (int)(4 * p->batch);
        return FFT_OK;
    }
    // rows pass -> tiled transpose -> rows pass (of the transposed grid) ->
    // tiled transpose back: for the long sides (> 2048) where the column
    // kernel's tiles get too narrow to stream (C4: 1.20 ms vs 1.40 ms)
    const char* tr_env = getenv("B200FFT_PIPE_TRANSPOSE");
    const bool tr_default = p->prec == 0 && N >= 256 && M >= 256 && (N > 2048 || M > 2048);
    if (filter == FFT_FILTER_GAUSS && !literal && (tr_env ? tr_env[0] == '1' : tr_default)) {
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        const size_t in_grid = (size_t)N * M * (real_in ? 4 : p->elem_bytes());
        const size_t grid = (size_t)N * M * p->elem_bytes();
        for (int64_t g = 0; g < p->batch; ++g) {
            char* o = (char*)out + g * grid;
            e = launch_rows(p->prec, false, real_in, M, (const char*)in + g * in_grid, o, N, 1.0 / (double)M, p->tw, st,
                            -1, -1, p->gv);
            if (e == cudaSuccess) e = launch_transpose(p->prec, o, p->ws, N, M, 1, st);
            if (e == cudaSuccess)
                e = launch_rows(p->prec, false, false, N, p->ws, p->ws, M, 1.0 / (double)N, p->tw, st, -1, -1, p->gu);
            if (e == cudaSuccess) e = launch_transpose(p->prec, p->ws, o, M, N, 1, st);
            if (e != cudaSuccess) return cuda_fail(e, "transposed pipeline launch");
        }
        p->last_launches = (int)(4 * p->batch);
        return FFT_OK;
    }
    if (filter == FFT_FILTER_GAUSS && !literal) {
        e = launch_rows(p->prec, false, real_in, M, in, out, p->batch * N, 1.0 / (double)M, p->tw, st, -1, -1,
                        p->gv);
        if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
        FilterArgs fc = f;
        fc.kind = 5;
        e = launch_cols(p->prec, 2, N, out, out, M, p->batch, 1.0 / (double)N, p->tw, fc, st);
        if (e != cudaSuccess) return cuda_fail(e, "k_cols launch");
        p->last_launches = 2;
        return FFT_OK;
    }
    e = launch_rows(p->prec, false, real_in, M, in, out, p->batch * N, 1.0, p->tw, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
    e = launch_cols(p->prec, 2, N, out, out, M, p->batch, 1.0 / ((double)N * (double)M), p->tw, f, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_cols launch");
    e = launch_rows(p->prec, true, false, M, out, out, p->batch * N, 1.0, p->tw, st);
    if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
    p->last_launches = 3;
    return FFT_OK;
}

// ---- distributed slab decomposition of rank-2 plans ---------------------
// P ranks (NCCL processes, or P virtual ranks on one GPU for tests).  Rank r
// owns rows [r SN, (r+1) SN) (SN = N/P) of every grid; after the first
// all-to-all it owns columns [r SM, (r+1) SM) (SM = M/P) as an [N][SM]
// row-major column slab.  Block q of a rank's send slab is its SN rows x the
// SM columns of rank q, which k_rows writes directly (blocked store), so the
// exchange needs no pack kernel; the way back lands blocked by source rank
// and k_rows reads it blocked (fused unpack).
//   pipeline: rows fwd -> a2a -> cols fwd*H/(NM)*inv -> a2a -> rows inv
//   forward : rows fwd -> a2a -> cols fwd (1/N) -> a2a -> unblock copy
//   inverse : rows inv (1/M) -> a2a -> cols inv -> a2a -> unblock copy
fft_status dist_exchange(fft_plan_s* p, char* send, char* recv, int64_t blk, cudaStream_t st) {
    const int P = p->P();
    const size_t eb = p->elem_bytes(), bytes = (size_t)blk * eb;
    if (p->multi()) {
        if (!p->comm) return fail(FFT_E_UNSUPPORTED, "host collectives: the peer-memory schedule only");
#ifdef B200FFT_WITH_NCCL
        ncclComm_t comm = (ncclComm_t)p->comm;
        const ncclDataType_t dt = p->prec == 0 ? ncclFloat : ncclDouble;
        const size_t count = 2 * (size_t)blk;
        ncclResult_t r = ncclGroupStart();
        for (int q = 0; q < P && r == ncclSuccess; ++q) {
            r = ncclSend(send + q * bytes, count, dt, q, comm, st);
            if (r == ncclSuccess) r = ncclRecv(recv + q * bytes, count, dt, q, comm, st);
        }
        ncclResult_t r2 = ncclGroupEnd();
        if (r != ncclSuccess || r2 != ncclSuccess)
            return fail(FFT_E_NCCL, std::string("all-to-all: ") + ncclGetErrorString(r != ncclSuccess ? r : r2));
        return FFT_OK;
#else
        return fail(FFT_E_UNSUPPORTED, "library built without NCCL");
#endif
    }
    // virtual ranks: slab r of send/recv at r * P * blk; recv[q][r] = send[r][q]
    for (int r = 0; r < P; ++r) {
        cudaError_t e = cudaMemcpy2DAsync(recv + r * bytes, P * bytes, send + (size_t)r * P * bytes, bytes, bytes,
                                          (size_t)P, cudaMemcpyDeviceToDevice, st);
        if (e != cudaSuccess) return cuda_fail(e, "virtual all-to-all");
    }
    return FFT_OK;
}

// Column step of the slab schedule on one column slab [N][SM] (global
// columns col_off ..): the Gaussian pipeline's fwd * H / (N M) * inv as the
// three four-step column passes (N = 64 N2, as on one GPU; pass B applies
// g_N[k1 + 64 k2] g_M[col_off + v], filter kind 7), else one k_cols launch
// over the N-long columns.
cudaError_t dist_columns(fft_plan_s* p, char* cs, int mode, const FilterArgs& f, int64_t col_off, int64_t SM,
                         cudaStream_t st, int* launches) {
    const int64_t N = p->n0, M = p->n1;
    const char* c4 = getenv("B200FFT_PIPE_COLS4");
    if (mode == 2 && f.kind == FFT_FILTER_GAUSS && p->prec == 0 && colfilt_supported(N, SM) &&
        !(c4 && c4[0] == '0')) {
        // the three column phases in one kernel, the slab's groups in L2
        *launches += 1;
        return colfilt(p, cs, SM, 1, 1.0 / ((double)N * (double)M), f.gv, col_off, st);
    }
    if (mode == 2 && f.kind == FFT_FILTER_GAUSS && p->prec == 0 && N >= 4096 && N <= 8192 && SM >= 16 &&
        !(c4 && c4[0] == '0')) {
        cudaError_t e = ensure_twl(p, N);
        if (e != cudaSuccess) return e;
        const int64_t N1 = 64, N2 = N / 64;
        FilterArgs fa{};
        fa.tw_l = p->twl;
        fa.tdiv = SM;
        FilterArgs fb{};
        fb.kind = 7;
        fb.gu = f.gu;
        fb.gv = f.gv;
        fb.n1 = N1;
        fb.col_off = col_off;
        e = launch_cols_fourstep(3, N1, cs, cs, N2 * SM, 1, 1.0, p->tw, fa, st);
        if (e == cudaSuccess)
            e = launch_cols_fourstep(2, N2, cs, cs, SM, N1, 1.0 / ((double)N * (double)M), p->tw, fb, st);
        if (e == cudaSuccess) e = launch_cols_fourstep(4, N1, cs, cs, N2 * SM, 1, 1.0, p->tw, fa, st);
        *launches += 3;
        return e;
    }
    FilterArgs fl = f;
    fl.col_off = col_off;
    const int cmode = mode == 2 ? 2 : mode;
    const double sc = mode == 2 ? 1.0 / ((double)N * (double)M) : (mode == 0 ? 1.0 / (double)N : 1.0);
    *launches += 1;
    return launch_cols(p->prec, cmode, N, cs, cs, SM, 1, sc, p->tw, fl, st);
}

// ---- fused all-to-alls: direct block stores / loads over peer memory ----
// The row pass of rank r stores block q of its rows straight into rank q's
// receive slab (at block position r), and the final row pass (or unblock
// copy) loads block q of its rows straight from rank q's column slab: no
// send buffer, no NCCL all-to-all, two stream-ordered barriers per grid.
// Receive slabs alternate between two phases, so a rank still reading the
// previous grid's slabs never races with the next grid's stores (those only
// start after the next grid's first barrier).  Virtual ranks run the same
// schedule with local slabs and no barriers.
#ifdef B200FFT_WITH_NCCL
void p2p_release(fft_plan_s* p) {
    for (int q = 0; q < kMaxBlocks; ++q) {
        if (p->peer_buf[q] && q != p->my_rank) cudaIpcCloseMemHandle(p->peer_buf[q]);
        p->peer_buf[q] = nullptr;
    }
    if (p->p2p_buf) cudaFree(p->p2p_buf);
    if (p->bar_buf) cudaFree(p->bar_buf);
    p->p2p_buf = p->bar_buf = nullptr;
}

// collective: every rank of the communicator calls it at the same point
fft_status p2p_prepare(fft_plan_s* p, cudaStream_t st) {
    if (p->p2p != 0) return FFT_OK;
    const int P = p->nranks, me = p->my_rank;
    ncclComm_t comm = (ncclComm_t)p->comm;
    const char* env = getenv("B200FFT_P2P");
    struct Rec {
        cudaIpcMemHandle_t h;
        int ok;
        int pad;
    };
    Rec mine{};
    int ok = !(env && env[0] == '0') && P <= kMaxBlocks;
    const size_t bytes = 2 * (size_t)p->elems() * p->elem_bytes();
    if (ok && cudaMalloc(&p->p2p_buf, bytes) != cudaSuccess) ok = 0;
    if (ok && cudaMalloc(&p->bar_buf, 16) != cudaSuccess) ok = 0;
    if (ok && cudaMemsetAsync(p->bar_buf, 0, 16, st) != cudaSuccess) ok = 0;
    if (ok && cudaIpcGetMemHandle(&mine.h, p->p2p_buf) != cudaSuccess) ok = 0;
    cudaGetLastError();
    mine.ok = ok;
    // the handshake buffer was allocated by fft_plan_set_comm, so no local
    // failure can make this rank skip the all-gather the others are in
    static_assert(sizeof(Rec) * (kMaxBlocks + 1) <= 4096, "handshake buffer");
    std::vector<Rec> all(P);
    char* d = (char*)p->ctl_buf;
    bool all_ok;
    if (!comm) {  // host collectives (tests)
        cudaError_t e = cudaStreamSynchronize(st);
        all_ok = p->hc_allgather(p->hc_ctx, &mine, all.data(), sizeof(Rec)) == 0 && e == cudaSuccess;
    } else {
        cudaError_t e = cudaMemcpyAsync(d + P * sizeof(Rec), &mine, sizeof(Rec), cudaMemcpyHostToDevice, st);
        ncclResult_t r = ncclAllGather(d + P * sizeof(Rec), d, sizeof(Rec), ncclChar, comm, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(all.data(), d, sizeof(Rec) * P, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        all_ok = e == cudaSuccess && r == ncclSuccess;
    }
    for (int q = 0; q < P && all_ok; ++q) all_ok = all[q].ok != 0;
    int opened = 1;
    if (all_ok) {
        for (int q = 0; q < P; ++q) {
            if (q == me) {
                p->peer_buf[q] = p->p2p_buf;
            } else if (cudaIpcOpenMemHandle(&p->peer_buf[q], all[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                p->peer_buf[q] = nullptr;
                opened = 0;
                cudaGetLastError();
            }
        }
        // every rank must have mapped every peer
        if (!comm) {
            std::vector<int> op(P);
            all_ok = p->hc_allgather(p->hc_ctx, &opened, op.data(), sizeof(int)) == 0;
            for (int q = 0; q < P && all_ok; ++q) all_ok = op[q] == 1;
        } else {
            int* f = reinterpret_cast<int*>(d);
            cudaError_t e = cudaMemcpyAsync(f, &opened, sizeof(int), cudaMemcpyHostToDevice, st);
            ncclResult_t r = ncclAllReduce(f, f, 1, ncclInt32, ncclMin, comm, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&opened, f, sizeof(int), cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            all_ok = e == cudaSuccess && r == ncclSuccess && opened == 1;
        }
    }
    if (!all_ok) p2p_release(p);
    p->p2p = all_ok ? 1 : -1;
    if (getenv("B200FFT_VERBOSE")) fprintf(stderr, "rank %d: fused peer all-to-alls %s\n", me, all_ok ? "on" : "off");
    return FFT_OK;
}

// asynchronous communicator errors (a failed peer, a broken connection)
// surface here, after each distributed call's work is enqueued
fft_status nccl_async_check(fft_plan_s* p) {
    if (!p->comm) return FFT_OK;
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError((ncclComm_t)p->comm, &ar);
    if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("ncclCommGetAsyncError: ") + ncclGetErrorString(r));
    if (ar != ncclSuccess && ar != ncclInProgress)
        return fail(FFT_E_NCCL, std::string("communicator error: ") + ncclGetErrorString(ar));
    return FFT_OK;
}

fft_status dist_barrier(fft_plan_s* p, cudaStream_t st) {
    if (!p->comm) {  // host collectives (tests): drain, then the host barrier
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "barrier");
        if (p->hc_barrier(p->hc_ctx) != 0) return fail(FFT_E_NCCL, "host barrier failed");
        return FFT_OK;
    }
    ncclResult_t r = ncclAllReduce(p->bar_buf, p->bar_buf, 1, ncclFloat, ncclSum, (ncclComm_t)p->comm, st);
    if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("barrier: ") + ncclGetErrorString(r));
    return FFT_OK;
}
#endif

// the fused schedule; returns FFT_E_UNSUPPORTED (nothing launched) when it
// does not apply, and the caller runs the all-to-all schedule
fft_status run_dist_2d_fused(fft_plan_s* p, const void* in, void* out, int mode, const FilterArgs& f,
                             cudaStream_t st) {
    const int P = p->P();
    const char* ex = getenv("B200FFT_DIST_EXCHANGE");
    if (P > kMaxBlocks || (ex && ex[0] == '1')) return FFT_E_UNSUPPORTED;
    const int64_t N = p->n0, M = p->n1, SN = N / P, SM = M / P;
    const size_t eb = p->elem_bytes();
    const int64_t slab = SN * M, blk = SN * SM;
    const int sh = ilog2(SM);
    const int nloc = p->multi() ? 1 : P;
    const int r0 = p->multi() ? p->my_rank : 0;
    char* vbase = nullptr;
    if (p->multi()) {
#ifdef B200FFT_WITH_NCCL
        fft_status s = p2p_prepare(p, st);
        if (s != FFT_OK) return s;
        if (p->p2p != 1) return FFT_E_UNSUPPORTED;
#else
        return FFT_E_UNSUPPORTED;
#endif
    } else {
        fft_status s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        vbase = (char*)p->ws;
    }
    const bool real_in = mode == 2 && (p->flags & FFT_IN_REAL_F32);
    const size_t in_eb = real_in ? 4 : eb;
    cudaError_t e;
    int launches = 0;
    for (int64_t g = 0; g < p->batch; ++g) {
        const int ph = (int)(p->dist_phase++ & 1);
        // rank q's receive (column) slab of this phase
        auto rslab = [&](int q) -> char* {
            return p->multi() ? (char*)p->peer_buf[q] + (size_t)ph * slab * eb
                           : vbase + ((size_t)ph * P + q) * slab * eb;
        };
        const char* gin = (const char*)in + (size_t)g * nloc * slab * in_eb;
        char* gout = (char*)out + (size_t)g * nloc * slab * eb;
        // 1. rows of every local slab, block q stored into rank q's column slab
        for (int l = 0; l < nloc; ++l) {
            BlockPtrs ob{};
            for (int q = 0; q < P; ++q) ob.p[q] = rslab(q) + (size_t)(r0 + l) * blk * eb;
            const double sc = mode == 1 ? 1.0 / (double)M : 1.0;
            e = launch_rows(p->prec, mode == 1, real_in, M, gin + (size_t)l * slab * in_eb, nullptr, SN, sc, p->tw, st,
                            -1, sh, nullptr, nullptr, &ob);
            if (e != cudaSuccess) return cuda_fail(e, "k_rows (peer-store) launch");
            ++launches;
        }
        prof_mark(p, st, "rows+exchange(peer stores)");
#ifdef B200FFT_WITH_NCCL
        if (p->multi()) {
            fft_status s = dist_barrier(p, st);
            if (s != FFT_OK) return s;
            prof_mark(p, st, "barrier");
        }
#endif
        // 2. columns (length N) of every local column slab [N][SM], in place
        for (int l = 0; l < nloc; ++l) {
            e = dist_columns(p, rslab(r0 + l), mode, f, (int64_t)(r0 + l) * SM, SM, st, &launches);
            if (e != cudaSuccess) return cuda_fail(e, "column step launch");
        }
        prof_mark(p, st, "columns");
#ifdef B200FFT_WITH_NCCL
        if (p->multi()) {
            fft_status s = dist_barrier(p, st);
            if (s != FFT_OK) return s;
            prof_mark(p, st, "barrier");
        }
#endif
        // 3. rows of every local slab, block q loaded from rank q's column slab
        for (int l = 0; l < nloc; ++l) {
            BlockPtrs ib{};
            for (int q = 0; q < P; ++q) ib.p[q] = rslab(q) + (size_t)(r0 + l) * blk * eb;
            char* dst = gout + (size_t)l * slab * eb;
            if (mode == 2) {
                e = launch_rows(p->prec, true, false, M, nullptr, dst, SN, 1.0, p->tw, st, sh, -1, nullptr, &ib, nullptr);
                ++launches;
            } else {
                e = cudaSuccess;
                for (int q = 0; q < P && e == cudaSuccess; ++q)
                    e = cudaMemcpy2DAsync(dst + (size_t)q * SM * eb, M * eb, ib.p[q], SM * eb, SM * eb, (size_t)SN,
                                          cudaMemcpyDefault, st);
            }
            if (e != cudaSuccess) return cuda_fail(e, "final row pass / unblock (peer loads)");
        }
        prof_mark(p, st, mode == 2 ? "exchange(peer loads)+rows" : "exchange(peer loads)");
    }
    p->last_launches = launches;
    return FFT_OK;
}

// mode 0: forward (eq5), 1: inverse (2D-IDFT), 2: filter pipeline
fft_status run_dist_2d(fft_plan_s* p, const void* in, void* out, int mode, fft_filter filter, double param,
                       cudaStream_t st) {
    const int P = p->P();
    const int64_t N = p->n0, M = p->n1, SN = N / P, SM = M / P;
    if (N % P || M % P || SN < 1 || SM < 1) return fail(FFT_E_INVALID_SIZE, "grid not divisible by the rank count");
    fft_status s = FFT_OK;
    const size_t eb = p->elem_bytes();
    const int64_t slab = SN * M;      // elements per rank per grid
    const int64_t blk = SN * SM;      // elements per (rank, peer) block
    const int sh = ilog2(SM);
    const int nloc = p->multi() ? 1 : P;  // slabs handled by this process
    const int r0 = p->multi() ? p->my_rank : 0;
    const bool real_in = mode == 2 && (p->flags & FFT_IN_REAL_F32);
    const size_t in_eb = real_in ? 4 : eb;
    FilterArgs f{};
    f.kind = mode == 2 ? (int)filter : 0;
    f.N = N;
    f.M = M;
    if (mode == 2 && filter == FFT_FILTER_GAUSS) {
        s = gauss_tables(p, param);
        if (s != FFT_OK) return s;
        f.gu = p->gu;
        f.gv = p->gv;
    } else if (mode == 2) {
        f.b2 = param * param;
    }
    s = run_dist_2d_fused(p, in, out, mode, f, st);
    if (s != FFT_E_UNSUPPORTED) return s;
    s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    char* ws0 = (char*)p->ws;
    char* ws1 = ws0 + (size_t)nloc * slab * eb;
    cudaError_t e;
    int launches = 0;
    for (int64_t g = 0; g < p->batch; ++g) {
        const char* gin = (const char*)in + (size_t)g * nloc * slab * in_eb;
        char* gout = (char*)out + (size_t)g * nloc * slab * eb;
        // 1. rows (length M) of every local slab, stored in peer blocks
        for (int l = 0; l < nloc; ++l) {
            const bool inv_rows = mode == 1;
            const double sc = mode == 1 ? 1.0 / (double)M : 1.0;
            e = launch_rows(p->prec, inv_rows, real_in, M, gin + (size_t)l * slab * in_eb, ws0 + (size_t)l * slab * eb,
                            SN, sc, p->tw, st, -1, sh);
            if (e != cudaSuccess) return cuda_fail(e, "k_rows launch");
            ++launches;
        }
        prof_mark(p, st, "rows");
        s = dist_exchange(p, ws0, ws1, blk, st);
        if (s != FFT_OK) return s;
        prof_mark(p, st, "exchange(all-to-all)");
        // 2. columns (length N) of every local column slab [N][SM]
        for (int l = 0; l < nloc; ++l) {
            e = dist_columns(p, ws1 + (size_t)l * slab * eb, mode, f, (int64_t)(r0 + l) * SM, SM, st, &launches);
            if (e != cudaSuccess) return cuda_fail(e, "column step launch");
        }
        prof_mark(p, st, "columns");
        s = dist_exchange(p, ws1, ws0, blk, st);
        if (s != FFT_OK) return s;
        prof_mark(p, st, "exchange(all-to-all)");
        // 3. back to natural row slabs
        for (int l = 0; l < nloc; ++l) {
            const char* src = ws0 + (size_t)l * slab * eb;
            char* dst = gout + (size_t)l * slab * eb;
            if (mode == 2) {
                e = launch_rows(p->prec, true, false, M, src, dst, SN, 1.0, p->tw, st, sh, -1);
                ++launches;
            } else {
                // block q (SN x SM, from rank q) holds columns [q SM, (q+1) SM):
                // its row x (at src + (q SN + x) SM) goes to dst + x M + q SM
                e = cudaSuccess;
                for (int q = 0; q < P && e == cudaSuccess; ++q)
                    e = cudaMemcpy2DAsync(dst + (size_t)q * SM * eb, M * eb, src + (size_t)q * blk * eb, SM * eb,
                                          SM * eb, (size_t)SN, cudaMemcpyDeviceToDevice, st);
            }
            if (e != cudaSuccess) return cuda_fail(e, "unblock");
        }
        prof_mark(p, st, mode == 2 ? "rows" : "unblock");
    }
    p->last_launches = launches;
    return FFT_OK;
}

// ---- distributed four-step 1D (one transform of n = N1 N2 over P ranks) ----
// Rank r owns x[r n/P, (r+1) n/P) = rows n2 in [r S2, (r+1) S2) of the view
// A[n2][n1] = x[n1 + N1 n2] (S2 = N2/P).  Four-step (as fft_c2.cuh):
//   (A) FFT over n2 for each n1, (T) * W_n^{n1 k2}, (B) FFT over n1 for each
//   k2, X[k2 + N2 k1].
// Schedule per rank: transpose (pack) -> a2a -> unpack to [S1][N2] -> (A)
// rows -> (T) -> transpose -> a2a -> unpack to [S2][N1] -> (B) rows (1/n) ->
// transpose -> a2a -> unpack: rank r ends with X[r n/P, (r+1) n/P)
// (natural order, three all-to-alls).
fft_status fs_prepare(fft_plan_s* p) {
    const int P = p->P();
    const int m = ilog2(p->n0);
    const int64_t N1 = (int64_t)1 << (m - m / 2), N2 = (int64_t)1 << (m / 2);
    if (N1 % P || N2 % P) return fail(FFT_E_INVALID_SIZE, "transform too small for the rank count");
    if (p->sub_a && p->fs1 == N1 && p->sub_a->batch == N1 / P && p->sub_b->batch == N2 / P) return FFT_OK;
    // first use, or the rank count changed (fft_plan_set_virtual_ranks): rebuild
    if (p->sub_a) fft_plan_destroy(p->sub_a);
    if (p->sub_b) fft_plan_destroy(p->sub_b);
    if (p->fta) cudaFree(p->fta);
    if (p->ftb) cudaFree(p->ftb);
    p->sub_a = p->sub_b = nullptr;
    p->fta = p->ftb = nullptr;
    p->fs1 = N1;
    p->fs2 = N2;
    fft_precision prec = p->prec == 0 ? FFT_C64 : FFT_C128;
    int64_t d2 = N2, d1 = N1;
    fft_status s = fft_plan_create_ex(&p->sub_a, &d2, 1, N1 / P, prec, 0);
    if (s == FFT_OK) s = fft_plan_create_ex(&p->sub_b, &d1, 1, N2 / P, prec, 0);
    if (s != FFT_OK) return s;
    p->sub_a->scale_override = 1.0;                       // (A) unnormalised
    p->sub_b->scale_override = 1.0 / (double)p->n0;       // the paper's 1/n, once
    p->fsh = (m + 1) / 2;
    std::vector<double> a, b;
    const int64_t na = (int64_t)1 << (m - p->fsh), nb = (int64_t)1 << p->fsh;
    a.resize(2 * na);
    b.resize(2 * nb);
    for (int64_t i = 0; i < na; ++i) {
        const double ang = -2.0 * M_PI * (double)((i << p->fsh) % p->n0) / (double)p->n0;
        a[2 * i] = std::cos(ang);
        a[2 * i + 1] = std::sin(ang);
    }
    for (int64_t i = 0; i < nb; ++i) {
        const double ang = -2.0 * M_PI * (double)i / (double)p->n0;
        b[2 * i] = std::cos(ang);
        b[2 * i + 1] = std::sin(ang);
    }
    cudaError_t e = upload(a, p->prec, &p->fta);
    if (e == cudaSuccess) e = upload(b, p->prec, &p->ftb);
    if (e != cudaSuccess) return cuda_fail(e, "four-step twiddle upload");
    return FFT_OK;
}

// [P][R][Cb] blocks (by source rank) -> [R][P * Cb] rows, for each local slab
cudaError_t unpack_blocks(char* dst, const char* src, int64_t R, int64_t Cb, int P, size_t eb, cudaStream_t st) {
    cudaError_t e = cudaSuccess;
    for (int q = 0; q < P && e == cudaSuccess; ++q)
        e = cudaMemcpy2DAsync(dst + (size_t)q * Cb * eb, (size_t)P * Cb * eb, src + (size_t)q * R * Cb * eb, Cb * eb,
                              Cb * eb, (size_t)R, cudaMemcpyDeviceToDevice, st);
    return e;
}

// ---- NEXT-2: the paper's parallel schedule (Sec. 4) ----------
// P = 2^l ranks, n = 2^m.  Rank q holds its branch, the cyclic subsequence
// x[q + P j] (the leaves of processor idproc), and transforms it
// (levels 1..m1 = m - l).  Then l rounds: with nproc_sup = S
// active ranks, ranks q in [S/2, S) send their vector to q - S/2 and stop
// (P:165-190); each receiver combines the two with one radix-2 level
// (k_tree_combine); S halves.  After the last round the MASTER (rank 0)
// holds X = (1/n) DFT(x) in natural order.  Virtual ranks: all P
// branches are slabs of one buffer and every round is one batched combine.
fft_status tree_prepare(fft_plan_s* p) {
    const int P = p->P();
    const int64_t n = p->n0, L = n / P;
    const int nloc = p->multi() ? 1 : P;
    if (!p->tree_sub || p->tree_sub->n0 != L || p->tree_sub->batch != nloc) {
        if (p->tree_sub) fft_plan_destroy(p->tree_sub);
        p->tree_sub = nullptr;
        int64_t d = L;
        fft_status s = fft_plan_create_ex(&p->tree_sub, &d, 1, nloc, p->prec == 0 ? FFT_C64 : FFT_C128, 0);
        if (s != FFT_OK) return s;
    }
    if (!p->tta) {
        const int m = ilog2(n);
        p->tsh = (m + 1) / 2;
        const int64_t na = (int64_t)1 << (m - p->tsh), nb = (int64_t)1 << p->tsh;
        std::vector<double> a(2 * na), b(2 * nb);
        for (int64_t i = 0; i < na; ++i) {
            const double ang = -2.0 * M_PI * (double)((i << p->tsh) % n) / (double)n;
            a[2 * i] = std::cos(ang);
            a[2 * i + 1] = std::sin(ang);
        }
        for (int64_t i = 0; i < nb; ++i) {
            const double ang = -2.0 * M_PI * (double)i / (double)n;
            b[2 * i] = std::cos(ang);
            b[2 * i + 1] = std::sin(ang);
        }
        cudaError_t e = upload(a, p->prec, &p->tta);
        if (e == cudaSuccess) e = upload(b, p->prec, &p->ttb);
        if (e != cudaSuccess) return cuda_fail(e, "tree twiddle upload");
    }
    // buffers: virtual ranks ping-pong two n-element grids; a rank of a
    // communicator needs its largest vector twice plus the received half
    const size_t eb = p->elem_bytes();
    size_t need;
    if (!p->multi()) {
        need = 2 * (size_t)n * eb;
    } else {
        int64_t mx = L;
        for (int S = P; S > 1; S /= 2)
            if (p->my_rank < S / 2) mx *= 2;
        need = (size_t)(2 * mx + mx / 2 + 1) * eb;
    }
    if (p->tws_bytes < need) {
        if (p->tws) cudaFree(p->tws);
        p->tws = nullptr;
        p->tws_bytes = 0;
        cudaError_t e = cudaMalloc(&p->tws, need);
        if (e != cudaSuccess) return cuda_fail(e, "tree buffers");
        p->tws_bytes = need;
    }
    return FFT_OK;
}

fft_status run_paper_tree(fft_plan_s* p, const void* in, void* out, cudaStream_t st) {
    fft_status s = tree_prepare(p);
    if (s != FFT_OK) return s;
    const int P = p->P();
    const int64_t n = p->n0;
    int64_t M = n / P;
    const size_t eb = p->elem_bytes();
    char* A = (char*)p->tws;
    char* B = A + (size_t)n * eb;  // virtual ranks; a communicator rank re-slices below
    int launches = 0;
    p->tree_sub->stream = st;
    if (!p->multi()) {
        // 1. every branch: P slabs of n/P, one batched forward (1/(n/P))
        s = run_1d(p->tree_sub, in, A, false, st);
        if (s != FFT_OK) return s;
        launches += p->tree_sub->last_launches;
        // 2. rounds: receivers q < S/2 combine slab q (E) and slab q + S/2 (O)
        for (int S = P; S > 1; S /= 2) {
            char* dst = (S == 2) ? (char*)out : B;
            cudaError_t e = launch_tree_combine(p->prec, A, A + (size_t)(S / 2) * M * eb, dst, M, S / 2, M, 2 * M,
                                                n / (2 * M), p->tta, p->ttb, p->tsh, st);
            if (e != cudaSuccess) return cuda_fail(e, "tree combine");
            ++launches;
            std::swap(A, B);
            M *= 2;
        }
        if (P == 1) {
            cudaError_t e = cudaMemcpyAsync(out, A, (size_t)n * eb, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "tree copy");
        }
        p->last_launches = launches;
        return FFT_OK;
    }
#ifdef B200FFT_WITH_NCCL
    if (!p->comm) return fail(FFT_E_UNSUPPORTED, "host collectives: no tree schedule");
    const int q = p->my_rank;
    int64_t mx = M;
    for (int S = P; S > 1; S /= 2)
        if (q < S / 2) mx *= 2;
    char* V = A;                            // this rank's vector (<= mx)
    char* W = A + (size_t)mx * eb;          // combine target (<= mx)
    char* Rb = A + (size_t)2 * mx * eb;     // received half (<= mx / 2)
    const bool final_here = (q == 0 && out != nullptr);
    s = run_1d(p->tree_sub, in, (P == 1 && final_here) ? out : V, false, st);
    if (s != FFT_OK) return s;
    launches += p->tree_sub->last_launches;
    ncclComm_t comm = (ncclComm_t)p->comm;
    const ncclDataType_t dt = p->prec == 0 ? ncclFloat : ncclDouble;
    for (int S = P; S > 1; S /= 2) {
        if (q >= S) break;  // already sent its vector
        const size_t count = 2 * (size_t)M;
        ncclResult_t r;
        if (q >= S / 2) {
            r = ncclSend(V, count, dt, q - S / 2, comm, st);
            if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("tree send: ") + ncclGetErrorString(r));
            break;
        }
        r = ncclRecv(Rb, count, dt, q + S / 2, comm, st);
        if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("tree recv: ") + ncclGetErrorString(r));
        char* dst = (S == 2 && final_here) ? (char*)out : W;
        cudaError_t e = launch_tree_combine(p->prec, V, Rb, dst, M, 1, M, 2 * M, n / (2 * M), p->tta, p->ttb, p->tsh,
                                            st);
        if (e != cudaSuccess) return cuda_fail(e, "tree combine");
        ++launches;
        std::swap(V, W);
        M *= 2;
    }
    if (P == 1 && final_here) {
        // branch FFT already wrote out
    }
    p->last_launches = launches;
    return FFT_OK;
#else
    (void)out;
    return fail(FFT_E_UNSUPPORTED, "library built without NCCL");
#endif
}

// Steps (A) + (T) of the distributed four-step on one local slab [S1][N2],
// in place: the sub-FFTs over n2, then W_n^{(row0 + i) k2} -- fused into the
// epilogue of the one-pass 32768-point kernel when that kernel runs them
// (complex64, N2 = 32768; B200FFT_NO_TWFUSE=1: not fused), else the separate
// k_twiddle4 pass.
fft_status run_1d_twiddled(fft_plan_s* p, void* a, bool inv, int64_t row0, cudaStream_t st, int* launches) {
    fft_plan_s* sa = p->sub_a;
    const char* nf = getenv("B200FFT_NO_TWFUSE");
    if (p->prec == 0 && sa->tw4 && sa->n0 == 32768 && !(nf && nf[0] == '1')) {
        sa->otw_a = p->fta;
        sa->otw_b = p->ftb;
        sa->otw_sh = p->fsh;
        sa->otw_row0 = row0;
    }
    fft_status s = run_1d(sa, a, a, inv, st);
    const bool fused = sa->otw_done;
    sa->otw_a = sa->otw_b = nullptr;
    sa->otw_done = false;
    if (s != FFT_OK) return s;
    *launches += sa->last_launches;
    if (!fused) {
        cudaError_t e = launch_twiddle4(p->prec, inv, a, sa->batch, p->fs2, row0, p->fta, p->ftb, p->fsh, st);
        if (e != cudaSuccess) return cuda_fail(e, "twiddle");
        ++*launches;
    }
    return FFT_OK;
}

// Fused form of the schedule below: each pack -> all-to-all -> unpack is ONE
// distributed-transpose launch (k_dist_transpose) whose stores go straight
// into the other ranks' receive slabs (peer memory) -- the last one pulls
// this rank's natural-order output from the other ranks' slabs instead, as
// the caller's output buffer is not mapped by the peers.  Two receive
// phases: A ([S1][N2] after the first transpose) and B ([S2][N1]).  A rank
// pushes into phase A only after the previous call's barrier 2 (all ranks
// done with their phase-A work) and into phase B only after this call's
// barrier 1 (all ranks done pulling from phase B in the previous call); the
// natural-order pull of step 5 reads the peers' phase-B slabs after their
// in-place (B) FFTs, so it follows barrier 3 -- three stream-ordered
// barriers per transform (two with FFT_OUT_TRANSPOSED, whose step 4 reads
// only the local slab).  Virtual ranks: one launch per transpose for all P
// ranks, no barriers.
fft_status run_dist_1d_fused(fft_plan_s* p, const void* in, void* out, bool inv, cudaStream_t st) {
    const int P = p->P();
    const char* ex = getenv("B200FFT_DIST_EXCHANGE");
    if (P > kMaxBlocks || (ex && ex[0] == '1')) return FFT_E_UNSUPPORTED;
    fft_status s = fs_prepare(p);
    if (s != FFT_OK) return s;
    char* vbase = nullptr;
    if (p->multi()) {
#ifdef B200FFT_WITH_NCCL
        s = p2p_prepare(p, st);
        if (s != FFT_OK) return s;
        if (p->p2p != 1) return FFT_E_UNSUPPORTED;
#else
        return FFT_E_UNSUPPORTED;
#endif
    } else {
        s = ensure_workspace(p);
        if (s != FFT_OK) return s;
        vbase = (char*)p->ws;
    }
    p->sub_a->stream = st;
    p->sub_b->stream = st;
    const int64_t N1 = p->fs1, N2 = p->fs2, S1 = N1 / P, S2 = N2 / P;
    const int64_t loc = p->n0 / P;
    const size_t eb = p->elem_bytes();
    const int nloc = p->multi() ? 1 : P;
    const int r0 = p->multi() ? p->my_rank : 0;
    auto buf = [&](int ph, int q) -> char* {
        return p->multi() ? (char*)p->peer_buf[q] + (size_t)ph * loc * eb : vbase + ((size_t)ph * P + q) * loc * eb;
    };
    auto local = [&](const void* base, int q) -> void* {  // rank q's slab of a caller buffer
        return p->multi() ? (q == p->my_rank ? const_cast<void*>(base) : nullptr)
                       : (char*)const_cast<void*>(base) + (size_t)q * loc * eb;
    };
    BlockPtrs bin{}, ba{}, bb{}, bout{};
    for (int q = 0; q < P; ++q) {
        bin.p[q] = local(in, q);
        ba.p[q] = buf(0, q);
        bb.p[q] = buf(1, q);
        bout.p[q] = local(out, q);
    }
    cudaError_t e;
    int launches = 0;
    // 1. x viewed as [N2][N1] (rank r: rows n2 in [r S2, ..)) -> phase A
    //    [N1][N2] slabs of S1 rows (row n1, n2 global); push own rows
    e = launch_dist_transpose(p->prec, bin, ba, S2, N1, S1, P, (int64_t)r0 * S2, nloc * S2, 0, N1, st);
    if (e != cudaSuccess) return cuda_fail(e, "distributed transpose 1");
    ++launches;
    prof_mark(p, st, "exchange 1 (transpose, peer stores)");
#ifdef B200FFT_WITH_NCCL
    if (p->multi()) {
        if ((s = dist_barrier(p, st)) != FFT_OK) return s;
        prof_mark(p, st, "barrier");
    }
#endif
    // 2. (A) FFT over n2 (unnormalised) and (T) the four-step twiddle
    for (int l = 0; l < nloc; ++l) {
        char* a = buf(0, r0 + l);
        s = run_1d_twiddled(p, a, inv, (int64_t)(r0 + l) * S1, st, &launches);
        if (s != FFT_OK) return s;
    }
    prof_mark(p, st, "FFT over n2 + twiddle");
    // 3. phase A [N1][N2] (rows n1) -> phase B [N2][N1] slabs of S2 rows; push
    e = launch_dist_transpose(p->prec, ba, bb, S1, N2, S2, P, (int64_t)r0 * S1, nloc * S1, 0, N2, st);
    if (e != cudaSuccess) return cuda_fail(e, "distributed transpose 2");
    ++launches;
    prof_mark(p, st, "exchange 2 (transpose, peer stores)");
#ifdef B200FFT_WITH_NCCL
    if (p->multi()) {
        if ((s = dist_barrier(p, st)) != FFT_OK) return s;
        prof_mark(p, st, "barrier");
    }
#endif
    // 4. (B) FFT over n1 with the paper's 1/n (forward): Z[k2][k1] = X[k2 + N2 k1]
    const bool transposed_out = !inv && (p->flags & FFT_OUT_TRANSPOSED);
    for (int l = 0; l < nloc; ++l) {
        char* b = buf(1, r0 + l);
        const double saved = p->sub_b->scale_override;
        if (inv) p->sub_b->scale_override = 1.0;
        s = run_1d(p->sub_b, b, transposed_out ? (char*)bout.p[r0 + l] : b, inv, st);
        p->sub_b->scale_override = saved;
        if (s != FFT_OK) return s;
        launches += p->sub_b->last_launches;
    }
    prof_mark(p, st, "FFT over n1");
    if (!transposed_out) {
#ifdef B200FFT_WITH_NCCL
        // every rank's (B) FFTs ran in place in its phase-B slab: they must
        // all be complete before this rank pulls from the peers' slabs
        if (p->multi()) {
            if ((s = dist_barrier(p, st)) != FFT_OK) return s;
            prof_mark(p, st, "barrier");
        }
#endif
        // 5. natural order: Z [N2][N1] -> X as [N1][N2] slabs of S1 rows
        //    (rank r: rows k1 in [r S1, ..) = X[r n/P, ..)); pull own rows
        e = launch_dist_transpose(p->prec, bb, bout, S2, N1, S1, P, 0, N2, (int64_t)r0 * S1, nloc * S1, st);
        if (e != cudaSuccess) return cuda_fail(e, "distributed transpose 3");
        ++launches;
        prof_mark(p, st, "exchange 3 (transpose, peer loads)");
    }
    p->last_launches = launches;
    return FFT_OK;
}

fft_status run_dist_1d(fft_plan_s* p, const void* in, void* out, bool inv, cudaStream_t st) {
    fft_status s = run_dist_1d_fused(p, in, out, inv, st);
    if (s != FFT_E_UNSUPPORTED) return s;
    s = fs_prepare(p);
    if (s == FFT_OK) s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    p->sub_a->stream = st;
    p->sub_b->stream = st;
    const int P = p->P();
    const int64_t N1 = p->fs1, N2 = p->fs2, S1 = N1 / P, S2 = N2 / P;
    const int64_t loc = p->n0 / P;  // elements per rank
    const size_t eb = p->elem_bytes();
    const int nloc = p->multi() ? 1 : P;
    const int r0 = p->multi() ? p->my_rank : 0;
    char* w0 = (char*)p->ws;
    char* w1 = w0 + (size_t)nloc * loc * eb;
    cudaError_t e;
    int launches = 0;
    auto slab = [&](const void* base, int l) { return (char*)base + (size_t)l * loc * eb; };
    // 1. pack: A[S2][N1] -> [N1][S2] (block q = columns n1 of rank q)
    e = launch_transpose(p->prec, in, w0, S2, N1, nloc, st);
    if (e != cudaSuccess) return cuda_fail(e, "transpose");
    ++launches;
    s = dist_exchange(p, w0, w1, S1 * S2, st);
    if (s != FFT_OK) return s;
    // 2. unpack to [S1][N2] (row n1, n2 = q S2 + local)
    for (int l = 0; l < nloc; ++l) {
        e = unpack_blocks(slab(w0, l), slab(w1, l), S1, S2, P, eb, st);
        if (e != cudaSuccess) return cuda_fail(e, "unpack");
    }
    // 3. (A) FFT over n2 (unnormalised) and (T) the four-step twiddle
    for (int l = 0; l < nloc; ++l) {
        s = run_1d_twiddled(p, slab(w0, l), inv, (int64_t)(r0 + l) * S1, st, &launches);
        if (s != FFT_OK) return s;
    }
    // 4. pack [S1][N2] -> [N2][S1] (block q = rows k2 of rank q), exchange, unpack to [S2][N1]
    e = launch_transpose(p->prec, w0, w1, S1, N2, nloc, st);
    if (e != cudaSuccess) return cuda_fail(e, "transpose");
    ++launches;
    s = dist_exchange(p, w1, w0, S1 * S2, st);
    if (s != FFT_OK) return s;
    for (int l = 0; l < nloc; ++l) {
        e = unpack_blocks(slab(w1, l), slab(w0, l), S2, S1, P, eb, st);
        if (e != cudaSuccess) return cuda_fail(e, "unpack");
    }
    // 5. (B) FFT over n1 with the paper's 1/n (forward): Z[k2 local][k1]
    for (int l = 0; l < nloc; ++l) {
        const double saved = p->sub_b->scale_override;
        if (inv) p->sub_b->scale_override = 1.0;
        s = run_1d(p->sub_b, slab(w1, l), slab(w1, l), inv, st);
        p->sub_b->scale_override = saved;
        if (s != FFT_OK) return s;
        launches += p->sub_b->last_launches;
    }
    // 6a. FFT_OUT_TRANSPOSED (forward only): keep Z[k2 local][k1] = X[k2 + N2 k1]
    //     for this rank's k2 range -- one all-to-all less
    if (!inv && (p->flags & FFT_OUT_TRANSPOSED)) {
        for (int l = 0; l < nloc; ++l) {
            e = cudaMemcpyAsync(slab(out, l), slab(w1, l), (size_t)loc * eb, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "copy out");
        }
        p->last_launches = launches;
        return FFT_OK;
    }
    // 6. natural order: pack [S2][N1] -> [N1][S2] (block q = k1 of rank q), exchange, unpack
    e = launch_transpose(p->prec, w1, w0, S2, N1, nloc, st);
    if (e != cudaSuccess) return cuda_fail(e, "transpose");
    ++launches;
    s = dist_exchange(p, w0, w1, S1 * S2, st);
    if (s != FFT_OK) return s;
    for (int l = 0; l < nloc; ++l) {
        e = unpack_blocks(slab(out, l), slab(w1, l), S1, S2, P, eb, st);
        if (e != cudaSuccess) return cuda_fail(e, "unpack");
    }
    p->last_launches = launches;
    return FFT_OK;
}

fft_status dist_check(fft_plan_s* p) {
#ifdef B200FFT_WITH_NCCL
    return nccl_async_check(p);
#else
    (void)p;
    return FFT_OK;
#endif
}

fft_status check_ptrs(fft_plan_s* p, const void* in, void* out, bool real_in) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (!in || !out) return fail(FFT_E_INVALID_ARG, "null data pointer");
    if (!aligned(in, real_in ? 4 : p->elem_bytes()) || !aligned(out, p->elem_bytes()))
        return fail(FFT_E_INVALID_ARG, "data pointer not aligned to the element size");
    return FFT_OK;
}

}  // namespace

extern "C" {

const char* fft_status_string(fft_status s) {
    switch (s) {
        case FFT_OK: return "FFT_OK";
        case FFT_E_INVALID_SIZE: return "FFT_E_INVALID_SIZE";
        case FFT_E_INVALID_ARG: return "FFT_E_INVALID_ARG";
        case FFT_E_UNSUPPORTED: return "FFT_E_UNSUPPORTED";
        case FFT_E_CUDA: return "FFT_E_CUDA";
        case FFT_E_NCCL: return "FFT_E_NCCL";
        case FFT_E_ALLOC: return "FFT_E_ALLOC";
        case FFT_E_STATE: return "FFT_E_STATE";
    }
    return "FFT_E_UNKNOWN";
}

const char* fft_last_error(void) { return g_last_error.c_str(); }

const char* fft_build_info(void) {
    return "libb200fft sm_100a (nvcc " B200FFT_STR(__CUDACC_VER_MAJOR__) "." B200FFT_STR(__CUDACC_VER_MINOR__) ")";
}

fft_status fft_plan_create_ex(fft_plan* out, const int64_t* dims, int rank, int64_t batch,
                              fft_precision prec, unsigned flags) {
    if (!out) return fail(FFT_E_INVALID_ARG, "null plan output pointer");
    *out = nullptr;
    if (!dims) return fail(FFT_E_INVALID_ARG, "null dims");
    if (rank != 1 && rank != 2) return fail(FFT_E_INVALID_ARG, "rank must be 1 or 2");
    if (prec != FFT_C64 && prec != FFT_C128) return fail(FFT_E_INVALID_ARG, "bad precision");
    if (batch < 0) return fail(FFT_E_INVALID_SIZE, "negative batch");
    if (flags & ~(unsigned)(FFT_IN_REAL_F32 | FFT_OUT_TRANSPOSED | FFT_OUT_REAL_F32))
        return fail(FFT_E_INVALID_ARG, "unknown flag");
    if ((flags & FFT_OUT_REAL_F32) && (rank != 2 || !(flags & FFT_IN_REAL_F32) || prec != FFT_C64))
        return fail(FFT_E_INVALID_ARG, "FFT_OUT_REAL_F32 needs a rank-2 complex64 plan with FFT_IN_REAL_F32");
    const int ip = (int)prec;
    for (int d = 0; d < rank; ++d)
        if (!is_pow2(dims[d])) return fail(FFT_E_INVALID_SIZE, "transform sizes must be powers of two >= 1");
    if (rank == 1) {
        const int64_t lim = ip == 0 ? ((int64_t)1 << 30) : ((int64_t)1 << 28);
        if (dims[0] > lim) return fail(FFT_E_INVALID_SIZE, "1D length over the limit");
        if (flags & FFT_IN_REAL_F32) return fail(FFT_E_INVALID_ARG, "FFT_IN_REAL_F32 applies to rank-2 plans");
    } else {
        if (dims[0] > kColsMax[ip] || dims[1] > kRowsMax)
            return fail(FFT_E_INVALID_SIZE, "2D side over the limit");
        if ((flags & FFT_IN_REAL_F32) && ip != 0) return fail(FFT_E_INVALID_ARG, "FFT_IN_REAL_F32 needs complex64");
    }
    fft_plan_s* p = new fft_plan_s();
    p->rank = rank;
    p->n0 = dims[0];
    p->n1 = rank == 2 ? dims[1] : 1;
    p->batch = batch;
    p->prec = ip;
    p->flags = flags;
    cudaError_t e = cudaGetDevice(&p->device);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "cudaGetDevice");
    }
    e = device_twiddles(p->device, ip, &p->tw);
    if (e == cudaSuccess) e = c2_upload_constants();
    if (e == cudaSuccess) e = big_upload_constants();
    if (e == cudaSuccess) e = colfilt_upload_constants();
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "twiddle table upload");
    }
    int cn1 = 0, cn2 = 0;
    const char* no_c2 = getenv("B200FFT_NO_C2");
    if (rank == 1 && p->n0 > kRowsMax && !(no_c2 && no_c2[0] == '1') && c2_supported(ip, p->n0, &cn1, &cn2)) {
        // W_N^{n1 k2}, [k2][n1]
        std::vector<double> t(2 * (size_t)p->n0);
        for (int64_t k2 = 0; k2 < cn2; ++k2)
            for (int64_t n1 = 0; n1 < cn1; ++n1) {
                const int64_t x = (n1 * k2) % p->n0;
                const double ang = -2.0 * M_PI * (double)x / (double)p->n0;
                t[2 * (k2 * cn1 + n1)] = std::cos(ang);
                t[2 * (k2 * cn1 + n1) + 1] = std::sin(ang);
            }
        c2_plan_acquire(p->device);
        p->c2_acq = true;
        e = upload(t, ip, &p->tw4);
        if (e != cudaSuccess) {
            fft_plan_destroy(p);
            return cuda_fail(e, "four-step twiddle upload");
        }
    } else if (rank == 1 && p->n0 > kRowsMax) {
        p->radices = split_radices(p->n0, ip);
        // pass i (span Ns, radix R): W_{Ns R}^{k r} = pa[r][k mod KLO] * pb[r][k / KLO]
        int64_t Ns = 1;
        for (size_t i = 0; i < p->radices.size(); ++i) {
            const int64_t R = p->radices[i];
            const int64_t klo = Ns < 1024 ? Ns : 1024, nhi = Ns / klo;
            p->klo_sh.push_back(ilog2(klo));
            void* da = nullptr;
            void* db = nullptr;
            if (Ns > 1) {
                std::vector<double> a(2 * (size_t)(R * klo)), bt(2 * (size_t)(R * nhi));
                const int64_t n = Ns * R;
                for (int64_t r = 0; r < R; ++r) {
                    for (int64_t k = 0; k < klo; ++k) {
                        const double ang = -2.0 * M_PI * (double)((r * k) % n) / (double)n;
                        a[2 * (r * klo + k)] = std::cos(ang);
                        a[2 * (r * klo + k) + 1] = std::sin(ang);
                    }
                    for (int64_t h = 0; h < nhi; ++h) {
                        const double ang = -2.0 * M_PI * (double)((r * h * klo) % n) / (double)n;
                        bt[2 * (r * nhi + h)] = std::cos(ang);
                        bt[2 * (r * nhi + h) + 1] = std::sin(ang);
                    }
                }
                e = upload(a, ip, &da);
                if (e == cudaSuccess && nhi > 1) e = upload(bt, ip, &db);
                if (e != cudaSuccess) {
                    p->pa.push_back(da);
                    p->pb.push_back(db);
                    fft_plan_destroy(p);
                    return cuda_fail(e, "pass twiddle upload");
                }
            }
            p->pa.push_back(da);
            p->pb.push_back(db);
            Ns *= R;
        }
    }
    *out = p;
    return FFT_OK;
}

fft_status fft_plan_create(fft_plan* out, int64_t n, int64_t batch, int rank) {
    int64_t dims[2] = {n, n};
    return fft_plan_create_ex(out, dims, rank, batch, FFT_C64, 0);
}

fft_status fft_plan_set_stream(fft_plan p, void* s) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    p->stream = (cudaStream_t)s;
    return FFT_OK;
}

size_t fft_plan_workspace_bytes(fft_plan p) { return p ? workspace_need(p) : 0; }

fft_status fft_plan_set_workspace(fft_plan p, void* ptr, size_t bytes) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (bytes < workspace_need(p)) return fail(FFT_E_INVALID_ARG, "workspace too small");
    if (!ptr && bytes) return fail(FFT_E_INVALID_ARG, "null workspace");
    if (p->ws_owned && p->ws) cudaFree(p->ws);
    p->ws = ptr;
    p->ws_bytes = bytes;
    p->ws_owned = false;
    return FFT_OK;
}

static fft_status exec_body(fft_plan p, const void* in, void* out, bool inv);
static fft_status exec(fft_plan p, const void* in, void* out, bool inv) {
    fft_status s = check_ptrs(p, in, out, false);
    if (s != FFT_OK) return s;
    if (p->elems() == 0) return FFT_OK;
    prof_begin(p, p->stream);
    s = exec_body(p, in, out, inv);
    if (s == FFT_OK && p->prof && p->pn == 1) prof_mark(p, p->stream, inv ? "inverse" : "forward");
    return s;
}

static fft_status exec_body(fft_plan p, const void* in, void* out, bool inv) {
    fft_status s;
    // rank 1 on several ranks: the batch is sharded (each rank's plan holds its
    // own rows), so the local schedule is the whole job -- no collective
    if (p->rank == 1 && !p->dist()) return run_1d(p, in, out, inv, p->stream);
    if (!p->dist()) return run_2d(p, in, out, inv, p->stream);
    s = p->rank == 1 ? run_dist_1d(p, in, out, inv, p->stream)
                     : run_dist_2d(p, in, out, inv ? 1 : 0, FFT_FILTER_NONE, 0.0, p->stream);
    return s == FFT_OK ? dist_check(p) : s;
}

fft_status fft_forward(fft_plan p, const void* in, void* out) {
    NvtxRange r("b200fft.forward");
    return exec(p, in, out, false);
}

fft_status fft_forward_paper_tree(fft_plan p, const void* in, void* out) {
    NvtxRange nvtx("b200fft.forward_paper_tree");
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (p->rank != 1 || p->batch != 1) return fail(FFT_E_INVALID_ARG, "the paper's schedule needs a single 1D transform");
    if (!in) return fail(FFT_E_INVALID_ARG, "null input");
    const int P = p->P();
    if (P < 1 || (P & (P - 1))) return fail(FFT_E_INVALID_SIZE, "the paper's schedule needs 2^l ranks");
    if (p->multi() && !p->comm) return fail(FFT_E_UNSUPPORTED, "host collectives: no tree schedule");
    if (p->n0 % P) return fail(FFT_E_INVALID_SIZE, "n must be a multiple of the rank count");
    const bool master = !p->multi() || p->my_rank == 0;
    if (master && !out) return fail(FFT_E_INVALID_ARG, "rank 0 needs an n-element output");
    if (!aligned(in, p->elem_bytes()) || (out && !aligned(out, p->elem_bytes())))
        return fail(FFT_E_INVALID_ARG, "data pointer not aligned to the element size");
    fft_status s = run_paper_tree(p, in, master ? out : nullptr, p->stream);
    return s == FFT_OK ? dist_check(p) : s;
}
fft_status fft_inverse(fft_plan p, const void* in, void* out) {
    NvtxRange r("b200fft.inverse");
    return exec(p, in, out, true);
}

static fft_status check_real(fft_plan p, const void* in, void* out, bool c2r) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (!in || !out) return fail(FFT_E_INVALID_ARG, "null data pointer");
    if (p->dist()) return fail(FFT_E_UNSUPPORTED, "real transforms of a distributed plan");
    const int64_t M = p->rank == 2 ? p->n1 : p->n0;
    if (M < 2) return fail(FFT_E_INVALID_SIZE, "real transforms need a row length >= 2");
    const size_t rb = p->prec == 0 ? 4 : 8;
    if (!aligned(c2r ? in : out, p->elem_bytes()) || !aligned(c2r ? out : in, rb))
        return fail(FFT_E_INVALID_ARG, "data pointer not aligned");
    if (in == out) return fail(FFT_E_INVALID_ARG, "real transforms are out of place");
    return FFT_OK;
}

fft_status fft_forward_r2c(fft_plan p, const void* in, void* out) {
    NvtxRange nvtx("b200fft.forward_r2c");
    fft_status s = check_real(p, in, out, false);
    if (s != FFT_OK) return s;
    if (p->elems() == 0) return FFT_OK;
    prof_begin(p, p->stream);
    s = run_r2c(p, in, out, p->stream);
    if (s == FFT_OK && p->prof && p->pn == 1) prof_mark(p, p->stream, "r2c");
    return s;
}

fft_status fft_inverse_c2r(fft_plan p, const void* in, void* out) {
    NvtxRange nvtx("b200fft.inverse_c2r");
    fft_status s = check_real(p, in, out, true);
    if (s != FFT_OK) return s;
    if (p->elems() == 0) return FFT_OK;
    prof_begin(p, p->stream);
    s = run_c2r(p, in, out, p->stream);
    if (s == FFT_OK && p->prof && p->pn == 1) prof_mark(p, p->stream, "c2r");
    return s;
}

fft_status fft2d_filter_pipeline(fft_plan p, const void* in, void* out, fft_filter filter, double param) {
    NvtxRange nvtx("b200fft.filter_pipeline");
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (p->rank != 2) return fail(FFT_E_INVALID_ARG, "fft2d_filter_pipeline needs a rank-2 plan");
    const bool real_in = (p->flags & FFT_IN_REAL_F32) != 0;
    fft_status s = check_ptrs(p, in, out, real_in);
    if (s != FFT_OK) return s;
    if (filter < FFT_FILTER_NONE || filter > FFT_FILTER_IDEAL_LOWPASS) return fail(FFT_E_INVALID_ARG, "unknown filter");
    if (filter == FFT_FILTER_GAUSS && !(param > 0.0)) return fail(FFT_E_INVALID_ARG, "Gaussian needs param > 0");
    if ((filter == FFT_FILTER_IDEAL_LITERAL || filter == FFT_FILTER_IDEAL_LOWPASS) && !(param >= 0.0))
        return fail(FFT_E_INVALID_ARG, "ideal filter needs radius >= 0");
    if (real_in && in == out) return fail(FFT_E_INVALID_ARG, "real input cannot alias the complex output");
    if (p->elems() == 0) return FFT_OK;
    if (p->dist() && (p->flags & FFT_OUT_REAL_F32))
        return fail(FFT_E_UNSUPPORTED, "real-output pipeline on a distributed plan");
    prof_begin(p, p->stream);
    if (p->dist()) {
        s = run_dist_2d(p, in, out, 2, filter, param, p->stream);
        return s == FFT_OK ? dist_check(p) : s;
    }
    s = run_pipeline(p, in, out, filter, param, p->stream);
    if (s == FFT_OK && p->prof && p->pn == 1) prof_mark(p, p->stream, "pipeline");
    return s;
}

fft_status fft2d_image_filter_u8(fft_plan p, const uint8_t* in, int64_t h, int64_t w, uint8_t* out,
                                 fft_filter filter, double param, int max_val, float* spectrum) {
    NvtxRange nvtx("b200fft.image_filter_u8");
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (p->rank != 2 || p->prec != FFT_C64) return fail(FFT_E_INVALID_ARG, "image filter needs a rank-2 complex64 plan");
    if (p->dist()) return fail(FFT_E_UNSUPPORTED, "image filter on a distributed plan");
    if (!in || !out) return fail(FFT_E_INVALID_ARG, "null image pointer");
    if (spectrum && !aligned(spectrum, 4)) return fail(FFT_E_INVALID_ARG, "misaligned spectrum pointer");
    if (h < 1 || w < 1 || h > p->n0 || w > p->n1)
        return fail(FFT_E_INVALID_SIZE, "image must be 1 <= h <= N, 1 <= w <= M of the plan");
    if (max_val < 1 || max_val > 255) return fail(FFT_E_INVALID_ARG, "max_val must be in [1, 255]");
    if (filter < FFT_FILTER_NONE || filter > FFT_FILTER_IDEAL_LOWPASS) return fail(FFT_E_INVALID_ARG, "unknown filter");
    if (filter == FFT_FILTER_GAUSS && !(param > 0.0)) return fail(FFT_E_INVALID_ARG, "Gaussian needs param > 0");
    if ((filter == FFT_FILTER_IDEAL_LITERAL || filter == FFT_FILTER_IDEAL_LOWPASS) && !(param >= 0.0))
        return fail(FFT_E_INVALID_ARG, "ideal filter needs radius >= 0");
    const int64_t N = p->n0, M = p->n1;
    fft_status s = ensure_workspace(p);
    if (s != FFT_OK) return s;
    FilterArgs f{};
    f.kind = (int)filter;
    f.N = N;
    f.M = M;
    if (filter == FFT_FILTER_GAUSS) {
        s = gauss_tables(p, param);
        if (s != FFT_OK) return s;
        f.gu = p->gu;
        f.gv = p->gv;
    } else if (filter == FFT_FILTER_IDEAL_LITERAL || filter == FFT_FILTER_IDEAL_LOWPASS) {
        f.b2 = param * param;
    }
    f.spec_scale = (float)(1.0 / (double)N);  // eq5's 1/N
    cudaStream_t st = p->stream;
    const int64_t img_px = h * w;
    PdlScope pdl;  // three short kernels: each starts under the previous one's tail (31.7 -> 27.7 us)
    for (int64_t g = 0; g < p->batch; ++g) {
        f.spec = spectrum ? spectrum + g * N * M : nullptr;
        // pad + promote + rows forward (unnormalised) -> ws; columns fwd -> |F| -> x H / (N M) -> inv;
        // rows inverse -> real, round, clamp, crop -> out
        cudaError_t e = launch_image_rows(false, M, in + g * img_px, p->ws, N, N, h, w, max_val, p->tw, st);
        if (e == cudaSuccess)
            e = launch_cols(p->prec, 2, N, p->ws, p->ws, M, 1, 1.0 / ((double)N * (double)M), p->tw, f, st);
        if (e == cudaSuccess)
            e = launch_image_rows(true, M, p->ws, out + g * img_px, N, N, h, w, max_val, p->tw, st);
        if (e != cudaSuccess) return cuda_fail(e, "image filter launch");
    }
    p->last_launches = (int)(3 * p->batch);
    return FFT_OK;
}

fft_status fft_execute_host(fft_plan p, int direction, const void* host_in, void* host_out, fft_filter filter,
                            double param) {
    NvtxRange nvtx("b200fft.execute_host");
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (!host_in || !host_out) return fail(FFT_E_INVALID_ARG, "null host pointer");
    if (direction == 0 && p->rank != 2) return fail(FFT_E_INVALID_ARG, "pipeline needs a rank-2 plan");
    if (direction < -1 || direction > 1) return fail(FFT_E_INVALID_ARG, "direction must be -1, 0 or +1");
    if (p->dist()) return fail(FFT_E_UNSUPPORTED, "host execution of a distributed plan");
    if (p->flags & FFT_OUT_REAL_F32) return fail(FFT_E_UNSUPPORTED, "host execution of a real-output plan");
    const int64_t total = p->elems();
    if (total == 0) return FFT_OK;
    const bool real_in = direction == 0 && (p->flags & FFT_IN_REAL_F32);
    const size_t eb = p->elem_bytes();
    const size_t in_eb = real_in ? 4 : eb;
    // rows per chunk: 1D plans are split over the batch (independent
    // transforms); 2D plans over the batch of grids.
    const int64_t unit = p->rank == 1 ? p->n0 : p->n0 * p->n1;  // elements per transform
    const int64_t units = p->batch;
    // chunk size (B200FFT_HOST_CHUNK_MB, default 64 MiB): small enough that the
    // pipeline fill (first H2D) and drain (last D2H) stay short, large
    // enough to keep the copy engines at full rate
    static const size_t target = [] {
        const char* v = getenv("B200FFT_HOST_CHUNK_MB");
        const long mb = v ? atol(v) : 64;
        return (size_t)(mb > 0 ? mb : 64) << 20;
    }();
    int64_t per = (int64_t)(target / (unit * eb));
    if (per < 1) per = 1;
    if (per > units) per = units;
    const size_t chunk_bytes = (size_t)(per * unit) * eb;
    cudaError_t e;
    if (p->hbuf_bytes < chunk_bytes) {
        for (int i = 0; i < fft_plan_s::kHS; ++i) {
            if (p->hbuf[i]) cudaFree(p->hbuf[i]);
            if (p->hbin[i]) cudaFree(p->hbin[i]);
            p->hbuf[i] = p->hbin[i] = nullptr;
        }
        p->hbuf_bytes = 0;
        for (int i = 0; i < fft_plan_s::kHS; ++i) {
            e = cudaMalloc(&p->hbuf[i], chunk_bytes);
            if (e == cudaSuccess) e = cudaMalloc(&p->hbin[i], chunk_bytes);
            if (e != cudaSuccess) return fail(FFT_E_ALLOC, "host-execution staging buffers");
        }
        p->hbuf_bytes = chunk_bytes;
    }
    for (int i = 0; i < fft_plan_s::kHS; ++i)
        if (!p->hstream[i]) {
            e = cudaStreamCreateWithFlags(&p->hstream[i], cudaStreamNonBlocking);
            if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
        }
    if (!p->hev) {
        e = cudaEventCreateWithFlags(&p->hev, cudaEventDisableTiming);
        for (int i = 0; i < fft_plan_s::kHS && e == cudaSuccess; ++i)
            e = cudaEventCreateWithFlags(&p->hcomp[i], cudaEventDisableTiming);
        if (e != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
    }
    // order after the work already queued on the plan stream
    e = cudaEventRecord(p->hev, p->stream);
    for (int i = 0; i < fft_plan_s::kHS && e == cudaSuccess; ++i) e = cudaStreamWaitEvent(p->hstream[i], p->hev, 0);
    if (e != cudaSuccess) return cuda_fail(e, "stream ordering");
    const int64_t saved_batch = p->batch;
    int launches = 0;
    fft_status s = FFT_OK;
    for (int64_t u0 = 0, c = 0; u0 < units && s == FFT_OK; u0 += per, ++c) {
        const int64_t nu = (units - u0) < per ? (units - u0) : per;
        const int hs = (int)(c % fft_plan_s::kHS);
        cudaStream_t st = p->hstream[hs];
        void* d = p->hbuf[hs];
        void* din = p->hbin[hs];
        e = cudaMemcpyAsync(din, (const char*)host_in + (size_t)(u0 * unit) * in_eb, (size_t)(nu * unit) * in_eb,
                            cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) {
            s = cuda_fail(e, "H2D copy");
            break;
        }
        // the chunks' computes share the plan's workspace (the C2 ring and
        // counters, the 2D intermediate grid, the pass ping-pong buffer):
        // chunk c's compute starts after chunk c - 1's; with three streams the
        // H2D copy of chunk c + 1 and the D2H copy of chunk c - 1 both run
        // under chunk c's compute (PCIe in both directions at once)
        if (c > 0) {
            e = cudaStreamWaitEvent(st, p->hcomp[(c - 1) % fft_plan_s::kHS], 0);
            if (e != cudaSuccess) {
                s = cuda_fail(e, "chunk ordering");
                break;
            }
        }
        p->batch = nu;
        if (direction == 0)
            s = run_pipeline(p, din, d, filter, param, st);
        else
            s = p->rank == 1 ? run_1d(p, din, d, direction < 0, st) : run_2d(p, din, d, direction < 0, st);
        launches += p->last_launches;
        p->batch = saved_batch;
        if (s != FFT_OK) break;
        e = cudaEventRecord(p->hcomp[hs], st);
        if (e != cudaSuccess) {
            s = cuda_fail(e, "chunk ordering");
            break;
        }
        e = cudaMemcpyAsync((char*)host_out + (size_t)(u0 * unit) * eb, d, (size_t)(nu * unit) * eb,
                            cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) s = cuda_fail(e, "D2H copy");
    }
    p->last_launches = launches;
    cudaError_t es = cudaSuccess;
    for (int i = 0; i < fft_plan_s::kHS; ++i) {
        cudaError_t ei = cudaStreamSynchronize(p->hstream[i]);
        if (es == cudaSuccess) es = ei;
    }
    if (s != FFT_OK) return s;
    if (es != cudaSuccess) return cuda_fail(es, "host execution");
    return FFT_OK;
}

fft_status fft_nccl_unique_id(unsigned char id[128]) {
    if (!id) return fail(FFT_E_INVALID_ARG, "null id buffer");
#ifdef B200FFT_WITH_NCCL
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    static_assert(sizeof(u) == 128, "ncclUniqueId size");
    memcpy(id, &u, 128);
    return FFT_OK;
#else
    return fail(FFT_E_UNSUPPORTED, "library built without NCCL");
#endif
}

fft_status fft_plan_set_comm(fft_plan p, const unsigned char id[128], int nranks, int my_rank) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (nranks < 1 || my_rank < 0 || my_rank >= nranks) return fail(FFT_E_INVALID_ARG, "bad rank / nranks");
    if (p->multi()) return fail(FFT_E_STATE, "plan already has a communicator");
    if (p->virt > 1) return fail(FFT_E_STATE, "plan emulates virtual ranks");
    if (p->rank == 2 && (p->n0 % nranks || p->n1 % nranks))
        return fail(FFT_E_INVALID_SIZE, "2D sides must be divisible by the rank count");
    if (!id) return fail(FFT_E_INVALID_ARG, "null unique id");
    if (p->rank == 1 && p->batch != 1) {  // batch-sharded: no collective on the data path
        p->nranks = nranks;
        p->my_rank = my_rank;
        return FFT_OK;
    }
    if (p->rank == 1 && ((int64_t)nranks * nranks > p->n0 || p->n0 % nranks))
        return fail(FFT_E_INVALID_SIZE, "1D four-step needs n >= nranks^2");
#ifdef B200FFT_WITH_NCCL
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t comm = nullptr;
    ncclResult_t r = ncclCommInitRank(&comm, nranks, u, my_rank);
    if (r != ncclSuccess) return fail(FFT_E_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    cudaError_t ce = cudaMalloc(&p->ctl_buf, 4096);
    if (ce != cudaSuccess) {
        p->ctl_buf = nullptr;
        ncclCommDestroy(comm);
        return fail(FFT_E_ALLOC, std::string("communicator handshake buffer: ") + cudaGetErrorString(ce));
    }
    p->comm = comm;
    p->nranks = nranks;
    p->my_rank = my_rank;
    if (p->ws_owned && p->ws) {  // slab-sized workspace from now on
        cudaFree(p->ws);
        p->ws = nullptr;
        p->ws_bytes = 0;
    }
    return FFT_OK;
#else
    return fail(FFT_E_UNSUPPORTED, "library built without NCCL");
#endif
}

fft_status fft_plan_set_host_collectives(fft_plan p, int nranks, int my_rank, fft_host_allgather_fn allgather,
                                        fft_host_barrier_fn barrier, void* ctx) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (!allgather || !barrier) return fail(FFT_E_INVALID_ARG, "null collective callback");
    if (nranks < 1 || my_rank < 0 || my_rank >= nranks) return fail(FFT_E_INVALID_ARG, "bad rank / nranks");
    if (p->multi()) return fail(FFT_E_STATE, "plan already has a communicator");
    if (p->virt > 1) return fail(FFT_E_STATE, "plan emulates virtual ranks");
    if (p->rank == 1 && p->batch != 1) return fail(FFT_E_INVALID_ARG, "batch-sharded plans need no collectives");
    if (p->rank == 2 && (p->n0 % nranks || p->n1 % nranks))
        return fail(FFT_E_INVALID_SIZE, "2D sides must be divisible by the rank count");
    if (p->rank == 1 && ((int64_t)nranks * nranks > p->n0 || p->n0 % nranks))
        return fail(FFT_E_INVALID_SIZE, "1D four-step needs n >= nranks^2");
    p->hc_allgather = allgather;
    p->hc_barrier = barrier;
    p->hc_ctx = ctx;
    p->nranks = nranks;
    p->my_rank = my_rank;
    if (p->ws_owned && p->ws) {  // slab-sized workspace from now on
        cudaFree(p->ws);
        p->ws = nullptr;
        p->ws_bytes = 0;
    }
    return FFT_OK;
}

fft_status fft_plan_set_virtual_ranks(fft_plan p, int nranks) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    if (p->rank != 2 && p->batch != 1)
        return fail(FFT_E_INVALID_ARG, "virtual ranks apply to rank-2 plans and single 1D transforms");
    if (p->multi()) return fail(FFT_E_STATE, "plan has a communicator");
    if (nranks < 1 || p->n0 % nranks || (p->rank == 2 && p->n1 % nranks))
        return fail(FFT_E_INVALID_SIZE, "sizes must be divisible by the rank count");
    p->virt = nranks;
    if (p->ws_owned && p->ws) {
        cudaFree(p->ws);
        p->ws = nullptr;
        p->ws_bytes = 0;
    }
    return FFT_OK;
}

int fft_plan_last_launch_count(fft_plan p) { return p ? p->last_launches : 0; }

fft_status fft_plan_set_profiling(fft_plan p, int on) {
    if (!p) return fail(FFT_E_INVALID_ARG, "null plan");
    p->prof = on != 0;
    p->pn = 0;
    return FFT_OK;
}

int fft_plan_phase_times(fft_plan p, float* ms, int max, char* labels, size_t labels_bytes) {
    if (!p || !p->prof || p->pn < 2) return 0;
    if (cudaEventSynchronize(p->pev[p->pn - 1]) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    const int n = p->pn - 1 < max ? p->pn - 1 : max;
    std::string all;
    for (int k = 0; k < n; ++k) {
        float t = 0.f;
        if (ms && cudaEventElapsedTime(&t, p->pev[k], p->pev[k + 1]) == cudaSuccess) ms[k] = t;
        if (k) all += ';';
        all += p->plab[k];
    }
    if (labels && labels_bytes) {
        const size_t c = all.size() < labels_bytes - 1 ? all.size() : labels_bytes - 1;
        memcpy(labels, all.data(), c);
        labels[c] = 0;
    }
    return n;
}

fft_status fft_plan_destroy(fft_plan p) {
    if (!p) return FFT_OK;
    cudaError_t e = cudaSuccess;
    if (p->tw4) cudaFree(p->tw4);
    if (p->c2_acq) c2_plan_release(p->device);
    if (p->gbar) cudaFree(p->gbar);
    if (p->twl) cudaFree(p->twl);
    if (p->rtw) cudaFree(p->rtw);
    if (p->cws) cudaFree(p->cws);
    if (p->big_twl) cudaFree(p->big_twl);
    if (p->big_hi) cudaFree(p->big_hi);
    if (p->big_lo) cudaFree(p->big_lo);
    if (p->fta) cudaFree(p->fta);
    if (p->ftb) cudaFree(p->ftb);
    if (p->tree_sub) fft_plan_destroy(p->tree_sub);
    if (p->tta) cudaFree(p->tta);
    if (p->ttb) cudaFree(p->ttb);
    if (p->tws) cudaFree(p->tws);
    if (p->sub_a) fft_plan_destroy(p->sub_a);
    if (p->sub_b) fft_plan_destroy(p->sub_b);
    for (void* q : p->pa)
        if (q) cudaFree(q);
    for (void* q : p->pb)
        if (q) cudaFree(q);
    if (p->gu) cudaFree(p->gu);
    if (p->gv) cudaFree(p->gv);
    if (p->ws_owned && p->ws) cudaFree(p->ws);
    for (int i = 0; i < fft_plan_s::kHS; ++i) {
        if (p->hbuf[i]) cudaFree(p->hbuf[i]);
        if (p->hbin[i]) cudaFree(p->hbin[i]);
        if (p->hstream[i]) cudaStreamDestroy(p->hstream[i]);
    }
    if (p->hev) cudaEventDestroy(p->hev);
    for (cudaEvent_t ev : p->pev) cudaEventDestroy(ev);
    for (int i = 0; i < fft_plan_s::kHS; ++i)
        if (p->hcomp[i]) cudaEventDestroy(p->hcomp[i]);
#ifdef B200FFT_WITH_NCCL
    p2p_release(p);
    if (p->ctl_buf) cudaFree(p->ctl_buf);
    if (p->comm) ncclCommDestroy((ncclComm_t)p->comm);
#endif
    e = cudaGetLastError();
    delete p;
    if (e != cudaSuccess) return cuda_fail(e, "pending CUDA error at destroy");
    return FFT_OK;
}

}  // extern "C"
