mkdir -p gpurun_out
python scripts/prof_small.py c4 > gpurun_out/prof_plain_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 2 -c 2 -o gpurun_out/prof_c4 python scripts/prof_small.py c4 > gpurun_out/ncu_c4.log 2>&1
echo c4=$?
python scripts/prof_small.py c5 > gpurun_out/prof_plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 3 -c 3 -o gpurun_out/prof_c5 python scripts/prof_small.py c5 > gpurun_out/ncu_c5.log 2>&1
echo c5=$?
python scripts/prof_small.py c2 > gpurun_out/prof_plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ -s 1 -c 1 -o gpurun_out/prof_c2 python scripts/prof_small.py c2 > gpurun_out/ncu_c2.log 2>&1
echo c2=$?
