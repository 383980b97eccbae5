mkdir -p gpurun_out
python scripts/time_c3.py > gpurun_out/l2d_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_2d${TAG}.csv python scripts/time_c3.py > gpurun_out/l2d_ncu.log 2>&1
echo $?
