#!/bin/bash
# knob sweeps after the constant-table change: C2 (D margin, ring margin), C5 (D, ring margin)
mkdir -p gpurun_out
: > gpurun_out/sweep.txt
for d in 4 8 12; do for r in 32 40 48; do
  echo "AB_D=$d AB_RING=$r" >> gpurun_out/sweep.txt
  B200FFT_AB_D=$d B200FFT_AB_RING=$r timeout 120 python scripts/time_c2.py 10 >> gpurun_out/sweep.txt 2>&1
done; done
for d in 4 6 8; do for r in 4 6 8; do
  echo "BIG_D=$d BIG_RING=$r" >> gpurun_out/sweep.txt
  B200FFT_BIG_D=$d B200FFT_BIG_RING=$r timeout 300 python scripts/time_c4c5.py C5 >> gpurun_out/sweep.txt 2>&1
done; done
