# k_big at 2 CTAs/SM x 3 stages (B200FFT_BIG_2X3 bits: 1 = pass 1, 2 = pass 2) vs 3 x 2
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
B200FFT_BIG_2X3=3 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c5_config" -p no:cacheprovider 2>&1 | tail -2 | head -1
for v in 0 1 2 3 0 1; do echo "2x3=$v $(B200FFT_BIG_2X3=$v timeout -s KILL 200 python scripts/time_c4c5.py C5 | tail -1)"; done
