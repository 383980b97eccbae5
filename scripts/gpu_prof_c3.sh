mkdir -p gpurun_out
python scripts/prof_small.py c3 > gpurun_out/prof_plain_c3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 1 -c 1 -o gpurun_out/prof_c3 python scripts/prof_small.py c3 > gpurun_out/ncu_c3.log 2>&1
echo c3=$?
