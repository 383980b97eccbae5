# the distributed four-step's outer twiddle fused into k_ab_st<32768> (B200FFT_NO_TWFUSE=1: separate pass)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 900 python -m pytest tests/test_dist.py tests/test_gpu_parity.py tests/test_gpu_ipc.py tests/test_gpu_graph.py -m gpu -q -x -k "four_step or c5 or 32768 or tree or processes or graph" -p no:cacheprovider 2>&1 | tail -3
for env in "" "B200FFT_NO_TWFUSE=1" "" "B200FFT_NO_TWFUSE=1"; do echo "TREE $env: $(env $env timeout -s KILL 600 python bench.py --config TREE --steps 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k: (v["ms"], v["launches"]) for k, v in d["schedules"].items()})')"; done
