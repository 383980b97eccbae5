# C2 dependency / ring margins on the current box (B200FFT_AB_D: D margin, B200FFT_AB_RING: ring margin)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for cfg in "8 40" "4 40" "12 40" "16 40" "8 32" "8 48" "12 48" "16 56" "8 40"; do
  set -- $cfg
  echo "D+$1 ring+$2: $(B200FFT_AB_D=$1 B200FFT_AB_RING=$2 timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1 | cut -c1-90)"
done
