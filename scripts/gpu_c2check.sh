# which box: C2 forward timing + the fabric microbenchmark
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
nvidia-smi --query-gpu=serial,clocks.max.sm --format=csv,noheader
for i in 1 2; do timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1 | cut -c1-100; done
