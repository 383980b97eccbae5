# Round-2 evidence: smoke, the GPU suite, the default bench line, the reference arm, ncu traffic of every config
mkdir -p gpurun_out
R=${ROUND:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${R}_build.log 2>&1 || { echo build failed; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke=$?
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 -p no:cacheprovider > gpurun_out/${R}_pytest.log 2>&1; echo pytest=$?
tail -3 gpurun_out/${R}_pytest.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench=$?
timeout 300 python bench.py --impl reference --steps 3 > gpurun_out/${R}_bench_ref.json 2>/dev/null; echo ref=$?
timeout 300 python bench.py --config TREE --steps 3 > gpurun_out/${R}_bench_tree.json 2>/dev/null; echo tree=$?
if [ -z "$NOTRAFFIC" ]; then bash scripts/gpu_traffic.sh > gpurun_out/${R}_traffic.log 2>&1; echo traffic=$?; cp profiles/r2_traffic.json gpurun_out/${R}_traffic.json; fi
