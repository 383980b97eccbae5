#!/bin/bash
# C2 X-store policy vs DRAM traffic (ncu metrics of one forward launch) and time
mkdir -p gpurun_out
: > gpurun_out/c2pol.txt
for x in 0 128 256; do
  echo "XOPTS=$x" >> gpurun_out/c2pol.txt
  B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x timeout 120 python scripts/time_c2.py 10 >> gpurun_out/c2pol.txt 2>&1
  B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x C2_BATCH=4096 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum \
     --clock-control none -k regex:k_ab -s 1 -c 1 python scripts/prof_small.py c2 2>&1 | grep -E "dram__|gpu__time|lts__" >> gpurun_out/c2pol.txt
done
