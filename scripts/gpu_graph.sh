python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_gpu_graph.py tests/test_gpu_parity.py tests/test_gpu_batched2d.py tests/test_gpu_real.py -m gpu -q -x -k "graph or c3 or pipeline or fused or real" -p no:cacheprovider 2>&1 | tail -4
timeout -s KILL 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('C2', d['roofline']['fwd_ms_avg'], d['roofline']['frac'])
for k in ('C1','NEXT1','C3'):
    e=d['extra'][k]; print(k, {x:e.get(x) for x in ('us_median','graph_us_median','graph_us_min','ms_median','graph_output_identical','roundtrip_rel_l2')})
"
