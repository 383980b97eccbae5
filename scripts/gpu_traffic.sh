# ncu DRAM bytes + duration of every kernel of one step per config -> profiles/r2_traffic.json
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null || exit 1
for c in ${CFGS:-C2 C3 C3_real C4 C4_real C5}; do
  python scripts/traffic_step.py $c > gpurun_out/traffic_plain_$c.log 2>&1 || { echo "plain $c failed"; tail -3 gpurun_out/traffic_plain_$c.log; continue; }
  ncu --profile-from-start off --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --clock-control none --csv --log-file gpurun_out/traffic_$c.csv python scripts/traffic_step.py $c > gpurun_out/traffic_ncu_$c.log 2>&1
  echo "$c rc=$?"
done
python scripts/traffic_json.py gpurun_out profiles/r2_traffic.json
