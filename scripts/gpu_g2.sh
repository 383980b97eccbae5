#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/g2.txt
for g in 2 3 2 3; do
  echo "ROWS_G2=$g" >> gpurun_out/g2.txt
  B200FFT_ROWS_G2=$g timeout 600 python scripts/time_c4c5.py C4 >> gpurun_out/g2.txt 2>&1
done
B200FFT_ROWS_G2=3 timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "c4_config or 2d_8192 or colfilt" >> gpurun_out/g2.txt 2>&1
B200FFT_ROWS_G2=3 ncu --metrics gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none -k regex:k_rows_tma_g -s 1 -c 1 python scripts/prof_small.py c4 2>&1 | grep -E "gpu__time|bank" >> gpurun_out/g2.txt
