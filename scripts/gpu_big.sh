#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/big.txt
for x in 2 6 10 2 10; do
  echo "BIG_XO=$x" >> gpurun_out/big.txt
  B200FFT_BIG_XO=$x ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:k_big -s 0 -c 2 python scripts/prof_small.py c5 2>&1 | grep -E "gpu__time|dram" >> gpurun_out/big.txt
done
