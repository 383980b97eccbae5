python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_batched2d.py -m gpu -q -x -k "graph or c3 or pipeline or fused" -p no:cacheprovider 2>&1 | tail -2
for i in 1 2 3; do timeout -s KILL 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C2 fwd', d['roofline']['fwd_ms_avg'], 'C3', d['extra']['C3']['ms_median'], d['extra']['C3']['ms_min'], 'C3_real', d['extra']['C3_real']['ms_median'])"; done
