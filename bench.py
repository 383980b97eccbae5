#!/usr/bin/env python
"""bench.py -- throughput of the paper's FFT hot path on B200 (see DESIGN.md
"Measurement").

Default workload (BASELINE.json configs[1], the metric's config, "C2"):
4096 independent complex64 transforms of N = 65536 (N(0,1) parts, seed 2).
One step = forward (1/N) + inverse over the whole batch.  Metric: GFLOP/s in
the 5 N log2 N convention (2 transforms per row per step), whole job.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C2|C3|C4|C5|C1] [--extra]

Multi-GPU (torchrun, one process per GPU): the C2 batch is sharded with no
collective (weak scaling: every rank transforms its own 4096 rows of the
global seeded input stream).  Timing: CUDA events on the plan stream,
barrier + synchronize on both sides, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import math
import os
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
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback


def hbm_peak():
    try:
        with open(PEAKS_PATH) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled through NVML every
    ~5 ms while the timed region runs (the same counters nvidia-smi reports
    as clocks.sm / clocks_event_reasons.*)."""

    REASONS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
               "sw_power_cap": 0x4, "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.mx = None
        self.ok = False

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.ok = False
        return self

    def _poll(self):
        nv = self.nv
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.samples.append((sm, rs))
            except Exception:
                pass
            time.sleep(0.005)

    def __exit__(self, *a):
        self.stop.set()
        if self.ok:
            self.t.join(timeout=2)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.mx, "reasons": ["unavailable"], "samples": 0}
        reasons = set()
        for _, rs in self.samples:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.mx,
                "reasons": sorted(reasons), "samples": len(self.samples), "source": "NVML, 5 ms poll"}


# ------------------------------------------------------------- distributed
def dist_init(n_gpus):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl" if _cuda_ok() else "gloo")
    return ws, rank, local


def _cuda_ok():
    import torch

    return torch.cuda.is_available()


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(ws, v: float) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist

    t = torch.tensor([v], dtype=torch.float64, device="cuda" if _cuda_ok() else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------- C2
def flops_1d(n, batch, transforms_per_row=2):
    return 5.0 * n * math.log2(n) * batch * transforms_per_row


def cpu_baseline_c2(n=65536, target_s=12.0):
    """The oracle as it stands, on this host's cores, on a bounded sample of
    the C2 workload (forward + inverse of the first rows)."""
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
    return {"value": round(gf, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
            "sample": f"{rows} of 4096 rows of C2 (N=65536), forward+inverse, fp64, {dt:.1f} s"}


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
    xd = xh.to(dev, non_blocking=True)
    yd = torch.empty_like(xd)
    zd = torch.empty_like(xd)
    plan = b.Plan((n,), batch=batch, precision=b.C64, stream=stream)
    ws_t = torch.empty(max(plan.workspace_bytes(), 1), dtype=torch.uint8, device=dev)
    if plan.workspace_bytes():
        plan.set_workspace(ws_t)
    torch.cuda.synchronize()

    def step():
        plan.forward(xd, yd)
        l1 = plan.last_launch_count()
        plan.inverse(yd, zd)
        return l1 + plan.last_launch_count()

    for _ in range(args.warmup):
        step()
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
    ms = start.elapsed_time(end)
    ms = allreduce_max(ws, ms)
    fwd_ms = [e[0].elapsed_time(e[1]) for e in ev]
    inv_ms = [e[1].elapsed_time(e[2]) for e in ev]
    ms_step = ms / args.steps
    value = flops_1d(n, batch * ws) / (ms_step / 1e3) / 1e9

    # roofline of the dominant call (the forward transform: its launches)
    peak, peak_kind = hbm_peak()
    alg_bytes = 16.0 * n * batch
    fwd_avg = statistics.mean(fwd_ms)
    achieved = alg_bytes / (fwd_avg / 1e3) / 1e9
    traffic = None
    tr_path = os.path.join(ROOT, "profiles", "c2_traffic.json")
    if os.path.exists(tr_path):
        try:
            traffic = json.load(open(tr_path)).get("dram_bytes_per_launch")
        except Exception:
            traffic = None

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
        dt = time.perf_counter() - t0
        dt = allreduce_max(ws, dt)
        # the e2e result must be the round trip of the input (rel-L2 over the
        # whole batch, on the device) -- else the e2e number is not reported
        zd.copy_(back_h)
        e2e_err = float(torch.linalg.vector_norm(zd - xd) / torch.linalg.vector_norm(xd))
        if not e2e_err <= 1e-5:
            raise RuntimeError(f"execute_host round trip rel-L2 {e2e_err:.3e} > 1e-5")
        e2e = {"value": round(flops_1d(n, batch * ws) * e2e_steps / dt / 1e9, 3), "unit": "GFLOP/s",
               "h2d_bytes_per_step": 2 * 8 * n * batch, "d2h_bytes_per_step": 2 * 8 * n * batch,
               "steps": e2e_steps, "timer": "host wall clock around synchronous execute_host",
               "roundtrip_rel_l2": e2e_err}
        plan.inverse(yd, zd)  # restore zd for the device spot check below
        torch.cuda.synchronize()
    err = float(torch.linalg.vector_norm(zd[:64] - xd[:64]) / torch.linalg.vector_norm(xd[:64]))
    res = {
        "metric": "FFT GFLOP/s (5N*log2N), forward(1/N)+inverse",
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
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic,
                     "kernel": "forward transform (all its launches)", "peak_source": peak_kind,
                     "alg_bytes_per_launch": alg_bytes,
                     "fwd_ms_avg": round(fwd_avg, 4), "inv_ms_avg": round(statistics.mean(inv_ms), 4)},
        "gpu_launches": launches,
        "e2e": e2e,
        "roundtrip_rel_l2_first64rows": err,
        "clocks": clk.summary(),
    }
    plan.destroy()
    return res


# ---------------------------------------------------------- extra configs
def bench_c3(args, local, real_out=False):
    """C3 (BASELINE configs[2]); real_out: the NEXT-3 real-to-real form of the
    same pipeline (float32 out, two real rows per complex line)."""
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
    for _ in range(3):
        plan.filter_pipeline(idev, out, b.FILTER_GAUSS, 0.1)
    times = []
    for _ in range(max(args.steps, 20)):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()  # cold L2: write 512 MiB (> 126 MB L2) on the plan stream, before the timed region
            s.record(stream)
            plan.filter_pipeline(idev, out, b.FILTER_GAUSS, 0.1)
            e.record(stream)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    warm = []  # warm L2 (reported separately): back-to-back reps, no flush
    for _ in range(max(args.steps, 20)):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s.record(stream)
            plan.filter_pipeline(idev, out, b.FILTER_GAUSS, 0.1)
            e.record(stream)
        torch.cuda.synchronize()
        warm.append(s.elapsed_time(e))
    med = statistics.median(times)
    n = 2048 * 2048
    gf = 2 * 5 * n * math.log2(n) / (med / 1e3) / 1e9
    peak, _ = hbm_peak()
    alg = (16.0 if real_out else 32.0) * n  # float32 in + out vs complex64
    plan.destroy()
    name = ("NEXT-3: C3's pipeline real-to-real (float32 in/out), cold L2" if real_out
            else "C3: 2048^2 sky image Gaussian pipeline (cold L2)")
    return {"workload": name, "ms_median": round(med, 4),
            "ms_min": round(min(times), 4), "GFLOP/s": round(gf, 1),
            "hbm_frac": round(alg / (med / 1e3) / 1e9 / peak, 4),
            "warm_l2_ms_median": round(statistics.median(warm), 4)}


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
    for _ in range(3):
        plan.image_filter_u8(idev, out, b.FILTER_IDEAL_LITERAL, 340.0, 255, spec)
    times = []
    for _ in range(max(args.steps, 20)):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            flush.zero_()
            s.record(stream)
            plan.image_filter_u8(idev, out, b.FILTER_IDEAL_LITERAL, 340.0, 255, spec)
            e.record(stream)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e))
    med = statistics.median(times)
    n = 512 * 512
    plan.destroy()
    return {"workload": "NEXT-1: 506x460 uint8 image -> pad 512^2 -> FFT2 -> Eq. filtro b=340 -> IFFT2 -> uint8 "
                        "(+ spectrum), cold L2", "us_median": round(med * 1e3, 2), "us_min": round(min(times) * 1e3, 2),
            "GFLOP/s": round(2 * 5 * n * math.log2(n) / (med / 1e3) / 1e9, 1), "launches": 3}


def bench_c1(args, local):
    import torch

    import paper_cs_0103001_b200 as b

    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)
    x = fixtures.complex_input(1024, fixtures.UNIFORM, seed=1, dtype=np.complex128)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.empty_like(xd)
    plan = b.Plan((1024,), batch=1, precision=b.C128, stream=stream)
    for _ in range(5):
        plan.forward(xd, yd)
        plan.inverse(yd, yd)
    torch.cuda.synchronize()
    times = []
    for _ in range(50):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        plan.forward(xd, yd)
        plan.inverse(yd, yd)
        e.record(stream)
        torch.cuda.synchronize()
        times.append(s.elapsed_time(e) * 1e3)
    plan.destroy()
    return {"workload": "C1: N=1024 complex128 forward+inverse (latency)",
            "us_median": round(statistics.median(times), 2), "us_min": round(min(times), 2)}


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
        "metric": "FFT GFLOP/s (5N*log2N), forward(1/N)+inverse",
        "value": round(val, 4), "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C2: BASELINE configs[1] (bounded sample: 32 of 4096 rows per step)",
                   "n": n, "rows_per_step": rows},
        "cpu_baseline": {"value": round(val, 4), "unit": "GFLOP/s", "cores": cores, "kind": "oracle",
                         "sample": f"{rows} rows x N=65536 forward+inverse per step"},
        "e2e": {"value": round(val, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def bench_sharded(args, ws, rank, local, cfg):
    """C4 (8192^2 Gaussian pipeline, row slabs) or C5 (one 2^30 transform,
    four-step) across the ranks: the library's NCCL path when ws > 1."""
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
        a2a_per_step, alg_bytes = 2, 32.0 * loc
        workload = "C4: 8192^2 complex64 Gaussian pipeline, row slabs, 2 all-to-alls"
    else:
        n = 1 << 30
        loc = n // ws
        x = np.empty(loc, np.complex64)
        fixtures.complex_input(loc, fixtures.NORMAL, seed=5, offset=rank * loc, out=x)
        plan = b.Plan((n,), batch=1, stream=stream)
        flops = 2 * 5.0 * n * math.log2(n)
        a2a_per_step, alg_bytes = 6, 32.0 * loc
        workload = "C5: N=2^30 complex64 forward(1/N)+inverse, four-step, 3 all-to-alls per direction"
    if ws > 1:
        uid = [b.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        plan.set_comm(uid[0], ws, rank)
    xd = torch.from_numpy(x).to(dev)
    yd = torch.empty_like(xd)
    zd = torch.empty_like(xd)

    def step():
        if cfg == "C4":
            plan.filter_pipeline(xd, yd, b.FILTER_GAUSS, 0.1)
            return plan.last_launch_count()
        plan.forward(xd, yd)
        l1 = plan.last_launch_count()
        plan.inverse(yd, zd)
        return l1 + plan.last_launch_count()

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
    ms = allreduce_max(ws, s.elapsed_time(e)) / args.steps
    peak, peak_kind = hbm_peak()
    nvl = 8.0 * loc * (ws - 1) / ws * a2a_per_step  # bytes each GPU sends per step
    res = {
        "metric": "FFT GFLOP/s (5N*log2N), sharded", "value": round(flops / (ms / 1e3) / 1e9, 3),
        "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "c64 (fp32 arithmetic)", "data": "synthetic (counter-based seeded)",
        "config": {"workload": workload, "parallelism": f"slabs x{ws}, NCCL all-to-all" if ws > 1 else "1 GPU"},
        "roofline": {"bound": "hbm" if ws == 1 else "nvlink", "hbm_achieved_GBps_per_gpu":
                     round(alg_bytes / (ms / 1e3) / 1e9, 1), "hbm_peak": peak, "peak_source": peak_kind,
                     "nvlink_bytes_per_gpu_per_step": nvl,
                     "nvlink_GBps_per_gpu": round(nvl / (ms / 1e3) / 1e9, 1) if ws > 1 else None,
                     "nvlink_peak_GBps": 900.0},
        "gpu_launches": launches, "clocks": clk.summary(),
    }
    plan.destroy()
    return res


def bench_tree(args, ws, rank, local):
    """NEXT-2: the paper's own parallel schedule (Sec. 4) against
    the library's all-to-all four-step, forward only, on C5's transform
    (n = 2^30 complex64).  ws > 1: one rank per GPU, NCCL send/recv rounds;
    ws == 1: P = 8 VIRTUAL ranks on one GPU (all ranks' work serialised on
    one device: the arithmetic and HBM cost of the schedule, not its
    multi-GPU wall time -- labelled so).  Branch inputs: i.i.d. N(0,1) blocks
    (a cyclic subsequence of an i.i.d. sequence is i.i.d.)."""
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
        ms = allreduce_max(ws, s.elapsed_time(e)) / args.steps
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--config", default="C2", choices=["C2", "C4", "C5", "TREE"],
                    help="C2 (default, the metric's config), the sharded C4 / C5, or TREE (NEXT-2: the "
                         "paper's parallel schedule vs the all-to-all four-step)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--extra", action="store_true", help="also time C1, C3 and NEXT-1 (rank 0)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    ws, rank, local = dist_init(args.gpus)
    if args.impl == "reference":
        res = reference_arm(args, ws, rank)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    if args.config != "C2":
        res = (bench_tree(args, ws, rank, local) if args.config == "TREE"
               else bench_sharded(args, ws, rank, local, args.config))
        if rank == 0:
            print(json.dumps(res), flush=True)
        if ws > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    res = bench_c2(args, ws, rank, local)
    if rank == 0:
        if ws == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline_c2()
        if args.extra:
            res["extra"] = {"C1": bench_c1(args, local), "C3": bench_c3(args, local),
                            "C3_real": bench_c3(args, local, real_out=True), "NEXT1": bench_next1(args, local)}
        print(json.dumps(res), flush=True)
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
