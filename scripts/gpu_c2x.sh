#!/bin/bash
# ncu --set full of the current C2 forward kernel + part-off timings
mkdir -p gpurun_out
: > gpurun_out/c2x.txt
for x in 0 8 64 72; do
  echo "st XOPTS=$x" >> gpurun_out/c2x.txt
  B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x timeout 120 python scripts/time_c2.py 10 >> gpurun_out/c2x.txt 2>&1
done
C2_BATCH=4096 python scripts/prof_small.py c2 > gpurun_out/prof_plain.log 2>&1 && \
C2_BATCH=4096 ncu --set full --clock-control none --import-source on -k regex:"k_ab" -s 1 -c 1 \
    -o gpurun_out/r2s2_c2_full python scripts/prof_small.py c2 > gpurun_out/ncu_full.log 2>&1
echo full=$? >> gpurun_out/c2x.txt
