mkdir -p gpurun_out
export C2_BATCH=${C2_BATCH:-1024}
for v in ${VARIANTS:-10}; do
  B200FFT_CLUSTER_VARIANT=$v python scripts/prof_small.py c2 > gpurun_out/prof_plain_v$v.log 2>&1 && \
  B200FFT_CLUSTER_VARIANT=$v ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_} -s ${SKIP:-1} -c 1 \
      -o gpurun_out/prof_cluster_v$v python scripts/prof_small.py c2 > gpurun_out/ncu_full_v$v.log 2>&1
  echo v$v=$?
done
