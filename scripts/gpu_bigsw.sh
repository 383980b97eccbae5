python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c5_config" -p no:cacheprovider 2>&1 | tail -2
for i in 1 2; do echo "$(timeout -s KILL 200 python scripts/time_c4c5.py C5 | tail -1)"; done
