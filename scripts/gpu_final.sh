# Round-end evidence: smoke, the GPU suite, every bench line
mkdir -p gpurun_out
R=${ROUND:-r1final}
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke=$?
timeout -s KILL 2400 python -m pytest tests -m gpu -q --timeout 900 --durations=15 -p no:cacheprovider > gpurun_out/${R}_pytest.log 2>&1; echo pytest=$?
timeout 600 python bench.py --extra > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench=$?
timeout 300 python bench.py --config C4 --steps 5 > gpurun_out/${R}_bench_c4.json 2>/dev/null; echo c4=$?
timeout 300 python bench.py --config C5 --steps 3 > gpurun_out/${R}_bench_c5.json 2>/dev/null; echo c5=$?
timeout 300 python bench.py --config TREE --steps 3 > gpurun_out/${R}_bench_tree.json 2>/dev/null; echo tree=$?
timeout 300 python bench.py --impl reference --steps 2 > gpurun_out/${R}_bench_ref.json 2>/dev/null; echo ref=$?
