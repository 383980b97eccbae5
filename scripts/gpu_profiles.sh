# Evidence for profiles/: the bench line, the ncu launch list of the bench
# command, and one ncu --set full capture of the dominant kernel (C2 forward,
# full batch).  Each ncu command runs only after the same command exited 0.
mkdir -p gpurun_out
R=${ROUND:-r1}
python bench.py --extra > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err; echo bench=$?
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${R}_bench_small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_bench.csv \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${R}_ncu_launches.log 2>&1
echo launches=$?
C2_BATCH=4096 python scripts/prof_small.py c2 > gpurun_out/${R}_prof_plain.log 2>&1 && \
C2_BATCH=4096 ncu --set full --clock-control none --import-source on -k regex:"k_cluster|k_ab" -s 1 -c 1 \
    -o gpurun_out/${R}_c2_full python scripts/prof_small.py c2 > gpurun_out/${R}_ncu_full.log 2>&1
echo full=$?
