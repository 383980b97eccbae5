# Round-2 session-2 evidence: the round script (smoke, pytest -m gpu, default
# bench line, reference arm, TREE line, ncu traffic of every config), the ncu
# launch list of the bench command, and ncu --set full of each config's hot kernels
export ROUND=${ROUND:-r2s2}
bash scripts/gpu_round2.sh
python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/${ROUND}_bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${ROUND}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/${ROUND}_ncu_launches.log 2>&1
echo launches=$?
bash scripts/gpu_prof_c3.sh
bash scripts/gpu_prof_c4c5.sh
