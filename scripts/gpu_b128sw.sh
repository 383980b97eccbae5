python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_dist.py tests/test_gpu_graph.py -m gpu -q -x -k "32768 or c5_shape or four_step or graph_1d" -p no:cacheprovider 2>&1 | tail -2
python - <<'PY'
import subprocess, sys
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
print(f'32768 x 32768 fwd {m:.4f} ms, {16.0 * n * batch / m / 1e6:.0f} GB/s')
"""
for _ in range(2):
    print(subprocess.run([sys.executable, "-c", code], capture_output=True, text=True).stdout.strip())
PY
echo "TREE: $(timeout -s KILL 600 python bench.py --config TREE --steps 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: v["ms"] for k, v in d["schedules"].items()})')"
