#!/usr/bin/env python
"""bench.py -- throughput of the paper's FFT hot path on B200 (DESIGN.md
"Measurement").

Default line = BASELINE.json configs[1] ("C2", the metric's config): 4096
independent complex64 transforms of N = 65536 per GPU (N(0,1) parts, seed 2);
one step = forward (1/N) + inverse over the batch; metric GFLOP/s in the
5 N log2 N convention (2 transforms per row per step), whole job.  The same
line carries, under "extra", every other config at P = 1 (N = 1: C1 latency,
the C3 pipeline and its real-to-real form, NEXT-1, C4 and C5), and at N > 1
the sharded C4 / C5 (row slabs / four-step over the ranks, the library's
NCCL + peer-memory exchange) with per-phase exchange timing and an NCCL
all-to-all reference at the same message size.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C2|C4|C5|TREE] [--no-extra] [--no-e2e]

--gpus N > 1 without torchrun re-executes itself under torch.distributed.run
with N ranks; under torchrun WORLD_SIZE must equal N.  Timing: CUDA events on
the plan's stream, barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import fixtures  # noqa: E402  (seeded inputs; no method arithmetic)

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r2_traffic.json")
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
NVLINK_PEAK_GBS = 770.0    # B200_PROFILING.md: measured peer copy per direction (900 nominal)
METRIC = "FFT GFLOP/s (5N*log2N), forward(1/N)+inverse"


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


def traffic(key):
    """ncu DRAM bytes (read + write) of a config's step / kernel from the
    committed capture (scripts/gpu_traffic.py -> profiles/r2_traffic.json)."""
    try:
        with open(TRAFFIC_PATH) as fh:
            return json.load(fh).get(key)
    except Exception:
        return None


def roofline(alg_bytes, ms, kernel, tkey):
    peak, kind = hbm_peak()
    achieved = alg_bytes / (ms / 1e3) / 1e9
    t = traffic(tkey)
    tb = t.get("dram_bytes") if isinstance(t, dict) else None
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": tb,
            "traffic_ratio": round(tb / alg_bytes, 3) if tb else None,
            "alg_bytes": alg_bytes, "kernel": kernel, "peak_source": kind,
            # also against the nominal 8 TB/s HBM3e figure
            "frac_of_nominal_8000": round(achieved / 8000.0, 4)}


# ------------------------------------------------------------------ clocks
_NVML = {}


def _nvml_handle(index):
    """NVML initialised once per process (nvmlInit is slow: it must not
    delay the sampler's first sample inside a short timed region)."""
    if index not in _NVML:
        import pynvml

        pynvml.nvmlInit()
        _NVML[index] = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(index))
    return _NVML[index]


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    ~2 ms while the timed region runs (the counters nvidia-smi reports as
    clocks.sm / clocks_event_reasons.*).  The sampler runs until the region's
    work has completed on the device (the caller synchronises inside the
    `with` block), and always takes at least 5 samples."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    # NVML reports a clock change ~100 ms after it happens (measured: C2's
    # kernels slow down under sw_power_cap ~40 ms into a back-to-back run,
    # NVML shows it ~100 ms later), so sampling continues for TAIL seconds
    # after the region: the reasons are those seen in the region and the tail;
    # the median clock is over the region's samples only.
    TAIL = 0.15

    def __init__(self, index: int, period: float = 0.002):
        self.index = index
        self.period = period
        self.samples = []
        self.tail = []
        self.stop = threading.Event()
        self.mx = None
        self.ok = False

    def __enter__(self):
        try:
            self.nv, self.h = _nvml_handle(self.index)
            self.mx = self.nv.nvmlDeviceGetMaxClockInfo(self.h, self.nv.NVML_CLOCK_SM)
            self.ok = True
            self.started = threading.Event()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            self.started.wait(1.0)
        except Exception:
            self.ok = False
        return self

    def _poll(self):
        nv = self.nv
        t_stop = None
        while True:
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                (self.tail if t_stop is not None else self.samples).append((sm, rs))
            except Exception:
                pass
            self.started.set()
            if self.stop.is_set() and t_stop is None and len(self.samples) >= 5:
                t_stop = time.perf_counter()
            if t_stop is not None and time.perf_counter() - t_stop >= self.TAIL:
                break
            time.sleep(self.period)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2 + self.TAIL)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": ["unavailable"], "samples": 0}
        reasons = set()
        for _, rs in self.samples + self.tail:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        out = {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.mx,
               "reasons": sorted(reasons), "samples": len(self.samples),
               "source": f"NVML, {self.period * 1e3:.0f} ms poll, reasons include a "
                         f"{self.TAIL * 1e3:.0f} ms tail (NVML lags ~100 ms)"}
        if self.tail:
            out["sm_mhz_tail_min"] = min(s for s, _ in self.tail)
        return out


# ------------------------------------------------------------- distributed
def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def torchrun(n, argv, timeout=None):
    """Run bench.py with `argv` under torch.distributed.run, n ranks.  With a
    timeout the job runs in its own process group, killed whole (launcher and
    ranks) when the timeout expires, so no rank keeps a GPU afterwards."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.abspath(__file__), *argv]
    if timeout is None:
        return subprocess.run(cmd, cwd=ROOT)
    proc = subprocess.Popen(cmd, cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                            start_new_session=True)
    try:
        out, err = proc.communicate(timeout=timeout)
    except subprocess.TimeoutExpired:
        import signal

        os.killpg(proc.pid, signal.SIGKILL)
        proc.communicate()
        raise
    return subprocess.CompletedProcess(cmd, proc.returncode, out, err)


# Dry run of the N > 1 code paths on ONE GPU (B200FFT_BENCH_SHARE_GPU=1):
# every rank on cuda:0, gloo instead of NCCL, and the sharded configs'
# collectives by host callbacks (fft_plan_set_host_collectives).  Checks the
# orchestration only -- ranks share one GPU, so its times mean nothing and
# its lines say so ("dry_run").
SHARE_GPU = os.environ.get("B200FFT_BENCH_SHARE_GPU") == "1"


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = 0 if SHARE_GPU else int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() and not SHARE_GPU else "gloo")
    return ws, rank, local


def dist_done(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce(ws, v: float, op="max") -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda" if torch.cuda.is_available() and not SHARE_GPU else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def flops_1d(n, batch, transforms_per_row=2):
    return 5.0 * n * math.log2(n) * batch * transforms_per_row


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def timed(stream, fn, reps, flush=None):
    """Per-rep CUDA-event times (ms) of fn() on `stream`.  Cold L2: before
    each rep, outside the timed region, a 512 MiB buffer (> 126 MB L2) is
    zeroed on the same stream and then a 256 MiB slice of it is read back,
    so L2 holds none of the config's data and none of the flush's dirty lines
    (whose write-back would otherwise land in the timed region: +2 us on
    C3).  All reps are enqueued back to back and synchronised once, so host
    jitter (e.g. the clock sampler's NVML calls) never idles the GPU inside a
    timed region."""
    import torch

    evs = []
    with torch.cuda.stream(stream):
        for _ in range(reps):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if flush is not None:
                flush.zero_()
                flush[: flush.numel() // 2].sum()
            s.record(stream)
            fn()
            e.record(stream)
            evs.append((s, e))
    torch.cuda.synchronize()
    return [s.elapsed_time(e) for s, e in evs]


# ------------------------------------------------------------------- C2
def cpu_baseline_c2(n=65536, target_s=12.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of
    the C2 workload (forward + inverse of the first rows); plus single-thread
    timings of C1 and of a 64-row C2 subset."""
    import oracle

    cores = oracle.num_threads()
    rows = 16
    while True:
        x = fixtures.complex_input(rows * n, fixtures.NORMAL, seed=2).reshape(rows, n)
        t0 = time.perf_counter()
        y = oracle.fft_batch(x)
        oracle.fft_batch(y, inverse=True)
        dt = time.perf_counter() - t0
        if dt >= target_s / 4 or rows >= 4096:
            break
        rows = min(4096, int(rows * max(2.0, (target_s / 4) / max(dt, 1e-3))))
    gf = flops_1d(n, rows) / dt / 1e9
    single = {}
    try:
        oracle.set_num_threads(1)
        x1 = fixtures.complex_input(1024, fixtures.UNIFORM, seed=1, dtype=np.complex128)
        reps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < 0.5:
            oracle.ifft(oracle.fft(x1))
            reps += 1
        single["C1_fwd_inv_us"] = round((time.perf_counter() - t0) / reps * 1e6, 2)
        x64 = fixtures.complex_input(64 * n, fixtures.NORMAL, seed=2).reshape(64, n)
        t0 = time.perf_counter()
        y = oracle.fft_batch(x64)
        oracle.fft_batch(y, inverse=True)
        d1 = time.perf_counter() - t0
        single["C2_64rows_GFLOPs"] = round(flops_1d(n, 64) / d1 / 1e9, 4)
        single["C2_64rows_s"] = round(d1, 3)
    finally:
        oracle.set_num_threads(cores)
    return {"value": round(gf, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} of 4096 rows of C2 (N=65536), forward+inverse, fp64, {dt:.1f} s",
            "cpu_model": cpu_model(), "single_thread": single}


def bench_c2(args, ws, rank, local):
    import torch

    import paper_cs_0103001_b200 as b

    n, batch = 65536, 4096
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    # rank r owns global rows [r*batch, (r+1)*batch) of the seeded stream (weak scaling)
    x = fixtures.complex_input(batch * n, fixtures.NORMAL, seed=2, offset=rank * batch * n)
    xh = torch.from_numpy(x.reshape(batch, n)).pin_memory()
    del x
    xd = xh.to(dev, non_blocking=True)
    yd = torch.empty_like(xd)
    zd = torch.empty_like(xd)
    plan = b.Plan((n,), batch=batch, precision=b.C64, stream=stream)
    ws_t = torch.empty(max(plan.workspace_bytes(), 1), dtype=torch.uint8, device=dev)
    if plan.workspace_bytes():
        plan.set_workspace(ws_t)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        plan.forward(xd, yd)
        plan.inverse(yd, zd)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        start.record(stream)
        for i in range(args.steps):
            ev[i][0].record(stream)
            plan.forward(xd, yd)
            launches += plan.last_launch_count()
            ev[i][1].record(stream)
            plan.inverse(yd, zd)
            launches += plan.last_launch_count()
            ev[i][2].record(stream)
        end.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    ms = allreduce(ws, start.elapsed_time(end))
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    inv_ms = [e[1].elapsed_time(e[2]) for e in ev]
    ms_step = ms / args.steps
    value = flops_1d(n, batch * ws) / (ms_step / 1e3) / 1e9
    fwd_avg = allreduce(ws, statistics.mean(fwd_ms))
    alg_bytes = 16.0 * n * batch
    rf = roofline(alg_bytes, fwd_avg, "k_ab_st (forward: one launch)", "C2_fwd_kernel")
    rf.update({"alg_bytes_per_launch": alg_bytes, "fwd_ms_avg": round(fwd_avg, 4),
               "inv_ms_avg": round(allreduce(ws, statistics.mean(inv_ms)), 4),
               "timer": "CUDA events on the launching stream around each launch, averaged over the timed steps"})
    err = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))

    # end to end through the public API on host buffers (pinned), H2D + D2H inside
    e2e = None
    if not args.no_e2e:
        out_h = torch.empty_like(xh).pin_memory()
        back_h = torch.empty_like(xh).pin_memory()
        plan.execute_host(+1, xh, out_h)
        torch.cuda.synchronize()
        barrier(ws)
        e2e_steps = max(1, min(args.steps, 3))
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            plan.execute_host(+1, xh, out_h)
            plan.execute_host(-1, out_h, back_h)
        dt = allreduce(ws, time.perf_counter() - t0)
        # the e2e result must be the round trip of the input (rel-L2 over the
        # whole batch, on the device) -- else no e2e number is reported
        zd.copy_(back_h)
        e2e_err = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))
        if not e2e_err <= 1e-5:
            raise RuntimeError(f"execute_host round trip rel-L2 {e2e_err:.3e} > 1e-5")
        e2e = {"value": round(flops_1d(n, batch * ws) * e2e_steps / dt / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 2 * 8 * n * batch, "d2h_bytes_per_step": 2 * 8 * n * batch,
               "steps": e2e_steps, "timer": "host wall clock around synchronous execute_host, max over ranks",
               "roundtrip_rel_l2": e2e_err}
        del out_h, back_h
    res = {
        "metric": METRIC,
        "value": round(value, 3),
        "unit": "GFLOP/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "c64 (fp32 arithmetic)",
        "data": "synthetic (counter-based seeded N(0,1), fixtures/gen.c)",
        "config": {"workload": "C2: BASELINE configs[1], 4096 x N=65536 complex64 per GPU, forward(1/N)+inverse",
                   "n": n, "batch_per_gpu": batch, "global_batch": batch * ws,
                   "parallelism": f"batch-sharded x{ws}, no collective",
                   "l2": "inputs 2 GiB per buffer >> 126 MB L2 (no flush needed)"},
        "roofline": rf,
        "gpu_launches": launches,
        "e2e": e2e,
        "roundtrip_rel_l2": err,
        "clocks": clk.summary(),
    }
    plan.destroy()
    del xd, yd, zd, ws_t, xh
    torch.cuda.empty_cache()
    return res


# ---------------------------------------------------------- extra configs
def graph_of(stream, fn):
    """fn() (library calls on `stream`) captured once into a CUDA graph."""
    import torch

    g = torch.cuda.CUDAGraph()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        fn()
    torch.cuda.synchronize()
    return g


def bench_c1(args, local):
    """C1 (BASELINE configs[0]): N = 1024 complex128 forward + inverse;
    latency-bound (32 KiB), reported in microseconds."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    x = fixtures.complex_input(1024, fixtures.UNIFORM, seed=1, dtype=np.complex128)
    xd = torch.from_numpy(x).to(dev)
    yd, zd = torch.empty_like(xd), torch.empty_like(xd)
    plan = b.Plan((1024,), batch=1, precision=b.C128, stream=stream)

    def step():
        plan.forward(xd, yd)
        plan.inverse(yd, zd)

    for _ in range(5):
        step()
    # the same two library calls captured once into a CUDA graph (the plan
    # launches on its own stream, which is the capture stream): replays pay
    # one graph launch instead of two kernel launches
    graph = graph_of(stream, step)
    with ClockSampler(local) as clk:
        ts = timed(stream, step, 400)
        gts = timed(stream, graph.replay, 400)
    zd.zero_()
    graph.replay()
    torch.cuda.synchronize()
    err = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))
    plan.destroy()
    return {"workload": "C1: BASELINE configs[0], N=1024 complex128 forward+inverse (latency, warm L2)",
            "us_median": round(statistics.median(ts) * 1e3, 2), "us_min": round(min(ts) * 1e3, 2),
            "graph_us_median": round(statistics.median(gts) * 1e3, 2), "graph_us_min": round(min(gts) * 1e3, 2),
            "roofline": {"bound": "latency", "note": "32 KiB per transform: launch latency, not bandwidth"},
            "launches": 2, "roundtrip_rel_l2": err, "roundtrip_from": "graph replay", "clocks": clk.summary()}


def bench_c3(args, local, real_out=False):
    """C3 (BASELINE configs[2]); real_out: the NEXT-3 real-to-real form of the
    same pipeline (float32 out).  Cold L2 (see `timed`)."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    img = fixtures.sky_image(2048, 2048, seed=3)
    idev = torch.from_numpy(img).to(dev)
    out = torch.empty((2048, 2048), dtype=torch.float32 if real_out else torch.complex64, device=dev)
    plan = b.Plan((2048, 2048), batch=1, precision=b.C64,
                  flags=b.IN_REAL_F32 | (b.OUT_REAL_F32 if real_out else 0), stream=stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        plan.filter_pipeline(idev, out, b.FILTER_GAUSS, 0.1)

    for _ in range(3):
        step()
    with ClockSampler(local) as clk:
        cold = timed(stream, step, 200, flush)
        warm = timed(stream, step, 100)
    med = statistics.median(cold)
    n = 2048 * 2048
    alg = (16.0 if real_out else 32.0) * n
    name = ("NEXT-3: C3's pipeline real-to-real (float32 in/out), cold L2" if real_out
            else "C3: BASELINE configs[2], 2048^2 sky image Gaussian pipeline, cold L2")
    res = {"workload": name, "ms_median": round(med, 4), "ms_min": round(min(cold), 4),
           "GFLOP/s": round(2 * 5 * n * math.log2(n) / (med / 1e3) / 1e9, 1),
           "roofline": roofline(alg, med, f"the pipeline's {plan.last_launch_count()} launches",
                                "C3_real" if real_out else "C3"),
           "warm_l2_ms_median": round(statistics.median(warm), 4), "launches": plan.last_launch_count(),
           "clocks": clk.summary()}
    plan.destroy()
    return res


def bench_next1(args, local):
    """SURVEY NEXT-1, the paper's own application (Sec. 6): an
    8-bit 506 x 460 image (synthetic stand-in for NGC5194) zero-padded to
    512^2 -> 2D FFT -> Eq. (filtro) b = 340 -> 2D IFFT -> real, round, clamp,
    crop to uint8, spectrum written; cold L2, latency per image."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    img = fixtures.sky_image_u8(506, 460, seed=6)
    idev = torch.from_numpy(img).to(dev)
    out = torch.empty_like(idev)
    spec = torch.empty((512, 512), dtype=torch.float32, device=dev)
    plan = b.Plan((512, 512), batch=1, precision=b.C64, stream=stream)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step():
        plan.image_filter_u8(idev, out, b.FILTER_IDEAL_LITERAL, 340.0, 255, spec)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ref = out.clone()
    graph = graph_of(stream, step)
    with ClockSampler(local) as clk:
        ts = timed(stream, step, 200, flush)
        gts = timed(stream, graph.replay, 200, flush)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    graph_same = bool(torch.equal(out, ref))
    med = statistics.median(ts)
    n = 512 * 512
    plan.destroy()
    return {"workload": "NEXT-1: 506x460 uint8 image -> pad 512^2 -> FFT2 -> Eq. filtro b=340 -> IFFT2 -> uint8 "
                        "(+ spectrum), cold L2", "us_median": round(med * 1e3, 2), "us_min": round(min(ts) * 1e3, 2),
            "graph_us_median": round(statistics.median(gts) * 1e3, 2), "graph_output_identical": graph_same,
            "GFLOP/s": round(2 * 5 * n * math.log2(n) / (med / 1e3) / 1e9, 1), "launches": 3,
            "roofline": {"bound": "latency", "note": "2 MiB complex grid: three launches of ~10 us"},
            "clocks": clk.summary()}


def bench_c4_single(args, local):
    """C4 (BASELINE configs[3]) at P = 1: 8192^2 complex64 U[-1,1] (seed 4),
    Gaussian pipeline (forward 2D FFT -> H -> inverse 2D FFT) on one GPU."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    N = 8192
    x = torch.from_numpy(fixtures.complex_input(N * N, fixtures.UNIFORM, seed=4).reshape(N, N)).to(dev)
    y = torch.empty_like(x)
    plan = b.Plan((N, N), stream=stream)

    def step():
        plan.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1)

    for _ in range(3):
        step()
    with ClockSampler(local) as clk:
        ts = timed(stream, step, max(args.steps, 40))
    med = statistics.median(ts)
    launches = plan.last_launch_count()
    plan.destroy()
    alg = 32.0 * N * N
    return {"workload": "C4: BASELINE configs[3] at P=1, 8192^2 complex64 Gaussian pipeline on one GPU "
                        "(no exchange)",
            "ms_median": round(med, 4), "ms_min": round(min(ts), 4),
            "GFLOP/s": round(2 * 5 * N * N * math.log2(N * N) / (med / 1e3) / 1e9, 1),
            "roofline": roofline(alg, med, f"the pipeline's {launches} launches", "C4"),
            "launches": launches, "l2": "512 MiB grid >> L2", "clocks": clk.summary()}


def bench_c4_real(args, local):
    """NEXT-3 at the C4 size: an 8192^2 float32 sky image -> Gaussian ->
    float32, through the half spectrum (R2C rows, columns fwd*H*inv over the
    4097 columns, C2R rows); 16 B/pt (float in + out for two transforms)."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    N = 8192
    x = torch.from_numpy(fixtures.sky_image(N, N, seed=4, nsrc=2000)).to(dev)
    y = torch.empty_like(x)
    plan = b.Plan((N, N), flags=b.IN_REAL_F32 | b.OUT_REAL_F32, stream=stream)

    def step():
        plan.filter_pipeline(x, y, b.FILTER_GAUSS, 0.1)

    for _ in range(3):
        step()
    with ClockSampler(local) as clk:
        ts = timed(stream, step, max(args.steps, 40))
    med = statistics.median(ts)
    launches = plan.last_launch_count()
    plan.destroy()
    return {"workload": "NEXT-3 at the C4 size: 8192^2 float32 image, Gaussian pipeline real-to-real through the "
                        "Hermitian half spectrum",
            "ms_median": round(med, 4), "ms_min": round(min(ts), 4),
            "GFLOP/s": round(2 * 5 * N * N * math.log2(N * N) / (med / 1e3) / 1e9, 1),
            "roofline": roofline(16.0 * N * N, med, f"the pipeline's {launches} launches", "C4_real"),
            "launches": launches, "clocks": clk.summary()}


def bench_c5_single(args, local):
    """C5 (BASELINE configs[4]) at P = 1: one N = 2^30 complex64 transform
    (N(0,1), seed 5), forward (1/N) + inverse, multi-pass on one GPU."""
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    n = 1 << 30
    x = np.empty(n, np.complex64)
    fixtures.complex_input(n, fixtures.NORMAL, seed=5, out=x)
    xd = torch.from_numpy(x).to(dev)
    del x
    yd, zd = torch.empty_like(xd), torch.empty_like(xd)
    plan = b.Plan((n,), batch=1, stream=stream)
    fl = []

    def step():
        plan.forward(xd, yd)
        fl.append(plan.last_launch_count())
        plan.inverse(yd, zd)

    for _ in range(3):
        step()
    with ClockSampler(local) as clk:
        ts = timed(stream, step, max(args.steps // 2, 8))
    med = statistics.median(ts)
    err = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))
    plan.destroy()
    del xd, yd, zd
    torch.cuda.empty_cache()
    alg = 2 * 16.0 * n
    return {"workload": f"C5: BASELINE configs[4] at P=1, N=2^30 complex64 forward(1/N)+inverse, "
                        f"{fl[-1]} global passes per direction on one GPU (no exchange)",
            "ms_median": round(med, 4), "ms_min": round(min(ts), 4),
            "GFLOP/s": round(2 * 5 * n * 30 / (med / 1e3) / 1e9, 1),
            "roofline": roofline(alg, med, f"{fl[-1]} pass launches per direction", "C5"),
            "launches_per_direction": fl[-1], "roundtrip_rel_l2": err, "clocks": clk.summary()}


# --------------------------------------------------------- sharded configs
def bench_sharded_cfg(args, ws, rank, local, cfg):
    """C4 (8192^2 Gaussian pipeline, row slabs) or C5 (one 2^30 transform,
    four-step) across the ranks: the library's NCCL / peer-memory schedule.
    Besides the step time: a profiled step's per-phase device times (the
    exchange phases give the NVLink rate), a forward -> inverse round trip
    check, and the NCCL all-to-all of the same bytes as a reference."""
    import torch
    import torch.distributed as dist

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    if cfg == "C4":
        N = 8192
        loc = N * N // ws
        x = fixtures.complex_input(loc, fixtures.UNIFORM, seed=4, offset=rank * loc)
        plan = b.Plan((N, N), stream=stream)
        flops = 2 * 5.0 * N * N * math.log2(N * N)
        n_exch = 2
        workload = f"C4: 8192^2 complex64 Gaussian pipeline, row slabs of {N // ws} rows x {ws}, 2 exchanges"
    else:
        n = 1 << 30
        loc = n // ws
        x = np.empty(loc, np.complex64)
        fixtures.complex_input(loc, fixtures.NORMAL, seed=5, offset=rank * loc, out=x)
        plan = b.Plan((n,), batch=1, stream=stream)
        flops = 2 * 5.0 * n * math.log2(n)
        n_exch = 6
        workload = (f"C5: N=2^30 complex64 forward(1/N)+inverse, four-step 32768 x 32768 over {ws} ranks, "
                    "3 exchanges per direction (natural order)")
    if ws > 1 and SHARE_GPU:
        def allgather(mine):
            parts = [None] * ws
            dist.all_gather_object(parts, mine)
            return parts

        plan.set_host_collectives(ws, rank, allgather, dist.barrier)
    elif ws > 1:
        uid = [b.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        plan.set_comm(uid[0], ws, rank)
    xd = torch.from_numpy(x).to(dev)
    del x
    yd, zd = torch.empty_like(xd), torch.empty_like(xd)

    def step():
        if cfg == "C4":
            plan.filter_pipeline(xd, yd, b.FILTER_GAUSS, 0.1)
            return plan.last_launch_count()
        plan.forward(xd, yd)
        nl = plan.last_launch_count()
        plan.inverse(yd, zd)
        return nl + plan.last_launch_count()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    with ClockSampler(local) as clk:
        s.record(stream)
        for _ in range(args.steps):
            launches += step()
        e.record(stream)
        torch.cuda.synchronize()
    barrier(ws)
    ms = allreduce(ws, s.elapsed_time(e)) / args.steps
    # one profiled step: per-phase device times, max over ranks per phase
    plan.set_profiling(True)
    if cfg == "C4":
        plan.filter_pipeline(xd, yd, b.FILTER_GAUSS, 0.1)
        phases = plan.phase_times()
    else:
        plan.forward(xd, yd)
        phases = plan.phase_times()
        plan.inverse(yd, zd)
        phases += plan.phase_times()
    plan.set_profiling(False)
    phases = [(lab, allreduce(ws, t)) for lab, t in phases]
    ex_ms = sum(t for lab, t in phases if "exchange" in lab)
    bar_ms = sum(t for lab, t in phases if lab == "barrier")
    # round trip through the plan (a property at any size)
    if cfg == "C4":
        plan.forward(xd, yd)
        plan.inverse(yd, zd)
    torch.cuda.synchronize()
    num = allreduce(ws, float(torch.sum((zd - xd).abs().double() ** 2)), "sum")
    den = allreduce(ws, float(torch.sum(xd.abs().double() ** 2)), "sum")
    rt = math.sqrt(num / den)
    plan.destroy()
    nvl = 8.0 * loc * (ws - 1) / ws * n_exch  # bytes each GPU sends per step
    peak, _ = hbm_peak()
    res = {"workload": workload, "n_gpus": ws, "ms_per_step": round(ms, 4),
           "GFLOP/s": round(flops / (ms / 1e3) / 1e9, 1), "scaling": "strong", "gpu_launches": launches,
           "hbm_achieved_GBps_per_gpu": round(32.0 * loc / (ms / 1e3) / 1e9, 1), "hbm_peak": peak,
           "phases_ms": [[lab, round(t, 4)] for lab, t in phases],
           "roundtrip_rel_l2": rt, "clocks": clk.summary()}
    if ws > 1:
        res["roofline"] = {"bound": "nvlink", "exchanged_bytes_per_gpu_per_step": nvl,
                           "exchange_ms": round(ex_ms, 4), "barrier_ms": round(bar_ms, 4),
                           "achieved": round(nvl / (ex_ms / 1e3) / 1e9, 1) if ex_ms > 0 else None,
                           "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                           "frac": round(nvl / (ex_ms / 1e3) / 1e9 / NVLINK_PEAK_GBS, 4) if ex_ms > 0 else None,
                           "step_GBps": round(nvl / (ms / 1e3) / 1e9, 1),
                           "note": "exchange_ms = device time of the phases that move data between GPUs "
                                   "(peer stores / loads fused into the row or transpose kernels)"}
    if ws > 1 and SHARE_GPU:
        res["dry_run"] = "ranks shared one GPU (B200FFT_BENCH_SHARE_GPU): times are not measurements"
    elif ws > 1:
        # NCCL all-to-all of one exchange's bytes (reference)
        t = torch.empty(2 * loc, dtype=torch.float32, device=dev)
        o = torch.empty_like(t)
        for _ in range(3):
            dist.all_to_all_single(o, t)
        torch.cuda.synchronize()
        barrier(ws)
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s2.record()
        for _ in range(5):
            dist.all_to_all_single(o, t)
        e2.record()
        torch.cuda.synchronize()
        a2a_ms = allreduce(ws, s2.elapsed_time(e2)) / 5
        one = 8.0 * loc * (ws - 1) / ws
        res["nccl_all_to_all"] = {"ms": round(a2a_ms, 4), "bytes_per_gpu": one,
                                  "GBps_per_gpu": round(one / (a2a_ms / 1e3) / 1e9, 1)}
        del t, o
    del xd, yd, zd
    torch.cuda.empty_cache()
    return res


def bench_tree(args, ws, rank, local):
    """NEXT-2: the paper's own parallel schedule (Sec. 4) against
    the library's all-to-all four-step, forward only, on C5's transform
    (n = 2^30 complex64).  ws > 1: one rank per GPU, NCCL send/recv rounds;
    ws == 1: P = 8 VIRTUAL ranks on one GPU (all ranks' work serialised on
    one device: the arithmetic and HBM cost of the schedule, not its
    multi-GPU wall time -- labelled so)."""
    import torch
    import torch.distributed as dist

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(device=dev)
    n = 1 << 30
    P = ws if ws > 1 else 8
    loc = n // ws
    x = np.empty(loc, np.complex64)
    fixtures.complex_input(loc, fixtures.NORMAL, seed=5, offset=rank * loc, out=x)
    xd = torch.from_numpy(x).to(dev)
    del x
    res = {}
    for sched in ("paper_tree", "four_step_a2a"):
        plan = b.Plan((n,), batch=1, stream=stream)
        if ws > 1:
            uid = [b.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            plan.set_comm(uid[0], ws, rank)
        else:
            plan.set_virtual_ranks(P)
        if sched == "paper_tree":
            yd = torch.empty(n if rank == 0 else 1, dtype=torch.complex64, device=dev)
            run = lambda: plan.forward_paper_tree(xd, yd if rank == 0 else None)  # noqa: E731
        else:
            yd = torch.empty_like(xd)
            run = lambda: plan.forward(xd, yd)  # noqa: E731
        for _ in range(args.warmup):
            run()
        torch.cuda.synchronize()
        barrier(ws)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for _ in range(args.steps):
            run()
        e.record(stream)
        torch.cuda.synchronize()
        barrier(ws)
        ms = allreduce(ws, s.elapsed_time(e)) / args.steps
        res[sched] = {"ms": round(ms, 3), "GFLOP/s": round(5.0 * n * 30 / (ms / 1e3) / 1e9, 1),
                      "launches": plan.last_launch_count()}
        plan.destroy()
        del yd
        torch.cuda.empty_cache()
    return {"metric": "FFT GFLOP/s (5N*log2N), forward only", "value": res["paper_tree"]["GFLOP/s"],
            "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": res["paper_tree"]["ms"], "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "c64 (fp32 arithmetic)", "data": "synthetic (counter-based seeded)",
            "config": {"workload": "NEXT-2: the paper's tree schedule vs the all-to-all four-step, n = 2^30",
                       "ranks": P, "emulated": ws == 1,
                       "parallelism": f"{P} virtual ranks on 1 GPU (work serialised)" if ws == 1
                       else f"{ws} GPUs, NCCL send/recv rounds"},
            "schedules": res}


def reference_arm(args, ws, rank):
    """--impl reference: the fp64 oracle (the paper's plain radix-2 tree) as it
    stands, on this host's cores, on a bounded sample of the C2 workload."""
    if rank != 0:
        return None
    import oracle

    n = 65536
    rows = 32
    cores = oracle.num_threads()
    x = fixtures.complex_input(rows * n, fixtures.NORMAL, seed=2).reshape(rows, n)
    for _ in range(args.warmup):
        oracle.fft_batch(x[:2])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        y = oracle.fft_batch(x)
        oracle.fft_batch(y, inverse=True)
    dt = (time.perf_counter() - t0) / args.steps
    val = flops_1d(n, rows) / dt / 1e9
    return {
        "impl": "reference",
        "metric": METRIC,
        "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: BASELINE configs[1] (bounded sample: 32 of 4096 rows per step)",
                   "n": n, "rows_per_step": rows},
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": f"{rows} rows x N=65536 forward+inverse per step", "cpu_model": cpu_model()},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _extra(name, fn, *a):
    try:
        return fn(*a)
    except Exception as ex:  # an extra config must not void the headline line
        return {"workload": name, "error": f"{type(ex).__name__}: {ex}"[:400]}


def sharded_extras(args, ws):
    """N > 1: the sharded C4 / C5 in a child torchrun job over the same GPUs
    (bounded by a 240 s timeout that kills the whole job, so a failure there
    can neither void the C2 line nor leave a rank holding a GPU)."""
    out = {}
    for cfg in ("C4", "C5"):
        try:
            r = torchrun(ws, ["--config", cfg, "--gpus", str(ws), "--steps", str(max(3, min(args.steps, 10))),
                              "--warmup", "3"], timeout=240)
            lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
            out[cfg] = json.loads(lines[-1]) if (r.returncode == 0 and lines) else \
                {"error": f"rc={r.returncode}: {r.stderr[-400:]}"}
        except subprocess.TimeoutExpired:
            out[cfg] = {"error": "timed out after 240 s (job killed)"}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--config", default="C2", choices=["C2", "C4", "C5", "TREE"],
                    help="C2 (default: the metric's config, with every other config under 'extra'), the "
                         "sharded C4 / C5 alone, or TREE (NEXT-2: the paper's parallel schedule vs the "
                         "all-to-all four-step)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extra", action="store_true", help="(the default now; kept for compatibility)")
    ap.add_argument("--no-extra", action="store_true", help="the C2 line only")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-execute under torch.distributed.run
        sys.exit(torchrun(args.gpus, sys.argv[1:]).returncode)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        print(f"bench.py: WORLD_SIZE={os.environ.get('WORLD_SIZE')} but --gpus {args.gpus}", file=sys.stderr)
        sys.exit(2)
    ws, rank, local = dist_init()
    if args.impl == "reference":
        res = reference_arm(args, ws, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        dist_done(ws)
        return
    if args.config != "C2":
        if args.config == "TREE":
            res = bench_tree(args, ws, rank, local)
        else:
            res = bench_sharded_cfg(args, ws, rank, local, args.config)
        if rank == 0:
            print(json.dumps(res), flush=True)
        dist_done(ws)
        return
    res = bench_c2(args, ws, rank, local)
    dist_done(ws)
    if rank == 0:
        if ws == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline_c2()
        if not args.no_extra:
            if ws == 1:
                res["extra"] = {"C1": _extra("C1", bench_c1, args, local),
                                "C3": _extra("C3", bench_c3, args, local),
                                "C3_real": _extra("C3_real", bench_c3, args, local, True),
                                "NEXT1": _extra("NEXT1", bench_next1, args, local),
                                "C4": _extra("C4", bench_c4_single, args, local),
                                "C4_real": _extra("C4_real", bench_c4_real, args, local),
                                "C5": _extra("C5", bench_c5_single, args, local)}
            else:
                res["extra"] = {"sharded": sharded_extras(args, ws)}
        if SHARE_GPU and ws > 1:
            res["dry_run"] = "ranks shared one GPU (B200FFT_BENCH_SHARE_GPU): times are not measurements"
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
