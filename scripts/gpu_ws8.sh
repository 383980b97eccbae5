# 8-line task pipeline (variants 45 / 46): parity, then timing against 44
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "c2_kernel" -p no:cacheprovider 2>&1 | tail -5
B200FFT_VERBOSE=1 timeout 200 python scripts/time_variants.py 44 45 46 44 2>&1 | grep -v "^persist" | tail -8
