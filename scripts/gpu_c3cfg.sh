#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/c3cfg.txt
for c in 0 1 2 0 1 2; do
  echo "ROWS2_CFG=$c" >> gpurun_out/c3cfg.txt
  B200FFT_ROWS2_CFG=$c timeout 300 python scripts/time_c3.py 2>&1 | head -1 >> gpurun_out/c3cfg.txt
done
for c in 1 2; do
B200FFT_ROWS2_CFG=$c timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_batched2d.py tests/test_gpu_parity.py -k "fused or c3_config or real_input" >> gpurun_out/c3cfg.txt 2>&1
done
