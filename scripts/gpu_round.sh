mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -12 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --extra --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?
cat gpurun_out/bench.json; tail -5 gpurun_out/bench.err
python scripts/prof_small.py all > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/prof_small.py all > gpurun_out/ncu_l.log 2>&1
echo ncu=$?
C2_BATCH=512 python scripts/prof_small.py c2 > gpurun_out/prof_plain2.log 2>&1 && \
C2_BATCH=512 ncu --set full --clock-control none --import-source on -k regex:k_cluster -s 1 -c 1 -o gpurun_out/prof_cluster python scripts/prof_small.py c2 > gpurun_out/ncu_full.log 2>&1
echo ncufull=$?
