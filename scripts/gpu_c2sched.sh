python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2" -p no:cacheprovider 2>&1 | tail -1
for x in 0 16 4 32 0; do
  echo "xo=$x: $(B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"
done
