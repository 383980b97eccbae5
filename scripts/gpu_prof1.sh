mkdir -p gpurun_out
python scripts/prof_small.py all > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches1.csv python scripts/prof_small.py all > gpurun_out/ncu_l.log 2>&1
C2_BATCH=512 python scripts/prof_small.py all > gpurun_out/prof_plain2.log 2>&1 && \
C2_BATCH=512 ncu --set full --clock-control none --import-source on -k regex:k_ -s 5 -c 5 -o gpurun_out/prof1 python scripts/prof_small.py all > gpurun_out/ncu_full.log 2>&1
echo done $?
