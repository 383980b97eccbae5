# k_ab_st<L = 32768>: parity, then 1D 32768 x 32768 timing vs the Stockham passes, TREE line (8 virtual ranks)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py -m gpu -q -x -k "32768 or multi_pass or c5 or four_step or tree or kernel_batches" -p no:cacheprovider 2>&1 | tail -3
python - <<'PY'
import os, statistics, subprocess, sys
code = r"""
import torch, statistics, sys
sys.path.insert(0, '.')
import paper_cs_0103001_b200 as b
n, batch = 32768, 32768
st = torch.cuda.Stream()
x = torch.randn(batch, n, dtype=torch.complex64, device='cuda')
y = torch.empty_like(x)
p = b.Plan((n,), batch=batch, stream=st)
for _ in range(3): p.forward(x, y)
torch.cuda.synchronize()
ts = []
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st); p.forward(x, y); e.record(st); torch.cuda.synchronize(); ts.append(s.elapsed_time(e))
m = statistics.median(ts)
print(f'{m:.4f} ms, {16.0 * n * batch / m / 1e6:.0f} GB/s, launches {p.last_launch_count()}')
"""
for env in ({}, {"B200FFT_NO_AB32K": "1"}, {}, {"B200FFT_NO_AB32K": "1"}):
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True, timeout=300)
    print("32768 x 32768 fwd", env or "k_ab_st<32768>", r.stdout.strip(), r.stderr[-300:] if r.returncode else "")
PY
for env in "" "B200FFT_NO_AB32K=1"; do echo "TREE $env: $(env $env timeout -s KILL 600 python bench.py --config TREE --steps 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: v["ms"] for k, v in d["schedules"].items()})')"; done
