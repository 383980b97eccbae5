# k_ab_pair (C2 with Y in TMEM, 2-CTA clusters): parity at small batches, then timing vs k_ab_st
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/pair_build.log 2>&1 || { echo build failed; tail gpurun_out/pair_build.log; exit 1; }
B200FFT_VERBOSE=1 timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "kernel_batches and pair" -p no:cacheprovider 2>&1 | tail -3
echo pytest=$?
for k in pair st; do B200FFT_C2=$k timeout -s KILL 120 python scripts/time_c2.py 10 2>&1 | tail -1; done
for xo in ${XOS:-1 2 4 8 16 64 3 5 72 95}; do echo "xo=$xo"; B200FFT_ALLOW_WRONG=1 B200FFT_PAIR_XO=$xo B200FFT_C2=pair timeout -s KILL 120 python scripts/time_c2.py 5 2>&1 | tail -1; done
