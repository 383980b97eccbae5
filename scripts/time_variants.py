"""Time the tuning variants of a plan (env knobs read at plan creation)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402


def time_plan(plan, x, y, reps=10):
    s = torch.cuda.current_stream()
    plan.set_stream(s)
    for _ in range(3):
        plan.forward(x, y)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record(s)
    for i in range(reps):
        plan.forward(x, y)
        ev[i + 1].record(s)
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]
    return min(ts), sorted(ts)[reps // 2]


def main():
    n, batch = 65536, int(os.environ.get("BATCH", "4096"))
    x = torch.from_numpy(fixtures.complex_input(batch * n, 1, seed=2).reshape(batch, n)).cuda()
    y = torch.empty_like(x)
    ref = None
    for var in sys.argv[1:] or ["0"]:
        os.environ["B200FFT_CLUSTER_VARIANT"] = var
        if var == "pass":
            os.environ["B200FFT_NO_CLUSTER"] = "1"
        p = b.Plan((n,), batch=batch)
        tmin, tmed = time_plan(p, x, y)
        os.environ.pop("B200FFT_NO_CLUSTER", None)
        out = y[:8].clone()
        err = 0.0 if ref is None else float((out - ref).abs().max() / ref.abs().max())
        ref = out if ref is None else ref
        gbs = 16.0 * n * batch / (tmed / 1e3) / 1e9
        print(f"variant {var}: min {tmin:.4f} ms  median {tmed:.4f} ms  {gbs:.0f} GB/s  "
              f"frac {gbs / 6554.6:.3f}  maxdiff-vs-first {err:.2e}", flush=True)
        p.destroy()


if __name__ == "__main__":
    main()
