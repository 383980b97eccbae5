# ncu --set full of this session's new kernels: k_ab_st<32768> and k_ab_pair (C2 with Y in TMEM)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python scripts/prof_small.py r32k > gpurun_out/prof_plain_r32k.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_ab_st -s 1 -c 1 -o gpurun_out/prof_r32k python scripts/prof_small.py r32k > gpurun_out/ncu_r32k.log 2>&1
echo r32k=$?
B200FFT_C2=pair python scripts/prof_small.py c2 > gpurun_out/prof_plain_pair.log 2>&1 && \
B200FFT_C2=pair ncu --set full --clock-control none --import-source on -k regex:k_ab_pair -s 1 -c 1 -o gpurun_out/prof_pair python scripts/prof_small.py c2 > gpurun_out/ncu_pair.log 2>&1
echo pair=$?
