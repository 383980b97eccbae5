mkdir -p gpurun_out
bash scripts/gpu_prof_c3.sh
python scripts/prof_small.py c4 > gpurun_out/prof_plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 2 -c 2 -o gpurun_out/prof_c4 python scripts/prof_small.py c4 > gpurun_out/ncu_c4.log 2>&1
echo c4=$?
