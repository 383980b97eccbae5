# fft_execute_host chunk size sweep (C2 e2e, PCIe-bound)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for c in 64 16 32 128 256 64; do B200FFT_HOST_CHUNK_MB=$c timeout -s KILL 300 python scripts/time_e2e.py | tail -1; done
