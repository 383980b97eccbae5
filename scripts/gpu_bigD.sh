# k_big phase distance / ring margin (groups) on the current box: C5 fwd + inv
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for cfg in ${CFGS:-"6 6" "4 6" "8 6" "6 4" "6 8" "5 6" "6 6"}; do
  set -- $cfg
  echo "D=$1 margin=$2: $(B200FFT_BIG_D=$1 B200FFT_BIG_RING=$2 timeout -s KILL 200 python scripts/time_c4c5.py C5 | tail -1)"
done
