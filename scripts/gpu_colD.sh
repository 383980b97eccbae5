# k_colfilt phase distance D (groups) on the current box: C4 pipeline time
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for d in ${DS:-32 24 32 24 32 24}; do echo "D=$d $(B200FFT_COLS1_D=$d timeout -s KILL 200 python scripts/time_c4c5.py C4 | tail -1)"; done
for d in 32 24; do echo "real D=$d $(B200FFT_COLS1_D=$d timeout -s KILL 200 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["extra"]["C4"]["ms_median"], d["extra"]["C4_real"]["ms_median"])')"; done
