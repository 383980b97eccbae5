"""C2 forward/inverse times per step over a long back-to-back run (does the
kernel slow down as the run goes on?), with NVML SM / memory clocks and power."""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import fixtures  # noqa: E402
import paper_cs_0103001_b200 as b  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
n, batch = 65536, 4096
st = torch.cuda.Stream()
p = b.Plan((n,), batch=batch, stream=st)
x = torch.from_numpy(fixtures.complex_input(batch * n, fixtures.NORMAL, seed=2).reshape(batch, n)).cuda()
y, z = torch.empty_like(x), torch.empty_like(x)
for _ in range(3):
    p.forward(x, y)
    p.inverse(y, z)
torch.cuda.synchronize()
samples = []
stop = False


def poll():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    while not stop:
        samples.append((time.perf_counter(), pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0,
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)))
        time.sleep(0.002)


th = threading.Thread(target=poll)
th.start()
ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
for i in range(steps):
    ev[i][0].record(st)
    p.forward(x, y)
    ev[i][1].record(st)
    p.inverse(y, z)
    ev[i][2].record(st)
torch.cuda.synchronize()
stop = True
th.join()
f = [e[0].elapsed_time(e[1]) for e in ev]
iv = [e[1].elapsed_time(e[2]) for e in ev]
for k in range(0, steps, 10):
    print(f"steps {k:3d}-{k + 9:3d}: fwd {sum(f[k:k + 10]) / 10:.4f} inv {sum(iv[k:k + 10]) / 10:.4f} ms")
if samples:
    for q in range(0, len(samples), max(1, len(samples) // 12)):
        t, sm, mem, pw, r = samples[q]
        print(f"  t={t - samples[0][0]:.3f}s sm {sm} mem {mem} power {pw:.0f} W reasons {r:#x}")
