# DRAM bytes and time of k_colfilt vs the phase distance D (C4 column pass)
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for d in ${DS:-8 16 24 32}; do
  B200FFT_COLS1_D=$d python scripts/traffic_step.py C4 > /dev/null 2>&1 && \
  B200FFT_COLS1_D=$d ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv -k regex:k_colfilt python scripts/traffic_step.py C4 2>/dev/null | grep k_colfilt | \
      awk -F'","' -v d=$d '{print "D=" d, $(NF-2), $(NF-1), $NF}'
done
