#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/big.txt
for gw in 16 32 16 32; do
  echo "GW2=$gw" >> gpurun_out/big.txt
  B200FFT_BIG_GW2=$gw ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none -k regex:k_big -s 1 -c 1 python scripts/prof_small.py c5 2>&1 | grep -E "k_big|gpu__time|dram" >> gpurun_out/big.txt
done
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "c5 or multi_pass" >> gpurun_out/big.txt 2>&1
B200FFT_BIG_GW2=16 timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py -k "c5" >> gpurun_out/big.txt 2>&1
python scripts/time_c4c5.py C5 >> gpurun_out/big.txt 2>&1
