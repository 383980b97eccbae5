# Parity + bench after a change: the GPU suite (or a subset), smoke, the default bench line
mkdir -p gpurun_out
R=${ROUND:-r2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${R}_build.log 2>&1 || { echo build failed; tail gpurun_out/${R}_build.log; exit 1; }
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo smoke=$?
timeout -s KILL ${PYT_TIMEOUT:-2400} python -m pytest ${TESTS:-tests} -m gpu -q -x --timeout 900 --durations=15 -p no:cacheprovider > gpurun_out/${R}_pytest.log 2>&1; echo pytest=$?
tail -25 gpurun_out/${R}_pytest.log
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench=$?
cat gpurun_out/${R}_bench.json; tail -5 gpurun_out/${R}_bench.err
fi
