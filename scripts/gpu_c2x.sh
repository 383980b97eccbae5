#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c2x.txt
for tw in 0 1 0 1; do
  echo "COLFILT_TW=$tw" >> gpurun_out/c2x.txt
  B200FFT_COLFILT_TW=$tw timeout 600 python scripts/time_c4c5.py C4 >> gpurun_out/c2x.txt 2>&1
done
