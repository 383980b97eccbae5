B200FFT_PASS_PIPE=5 timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider -k "multi_pass or three_pass or 65536_multipass" 2>&1 | tail -2
for v in 0 5; do echo "pipe=$v"; B200FFT_PASS_PIPE=$v python scripts/time_1d.py 20 24 27 30; B200FFT_PASS_PIPE=$v B200FFT_PASS_RMAX=8 python scripts/time_1d.py 30; done
