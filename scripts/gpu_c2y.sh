# C2 cache-hint A/B: 16384 = Y stores without a hint, 65536 = A loads without a hint
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for i in 1 2 3; do
for x in 0 16384 65536 81920; do
  echo "xo=$x: $(B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"
done; done
