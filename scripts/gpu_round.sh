mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -12 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --extra > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 300 python bench.py --config C4 --steps 5 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo c4=$?
cat gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
timeout 300 python bench.py --config C5 --steps 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
cat gpurun_out/bench_c5.json; tail -3 gpurun_out/bench_c5.err
timeout 300 python bench.py --impl reference --steps 2 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?
cat gpurun_out/bench_ref.json
