#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c2x.txt
for x in 0 1 2 3; do
  echo "ROWS_XO=$x" >> gpurun_out/c2x.txt
  B200FFT_ALLOW_WRONG=1 B200FFT_ROWS_XO=$x timeout 300 python scripts/time_c3.py >> gpurun_out/c2x.txt 2>&1
done
