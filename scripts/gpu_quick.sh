# quick GPU check: parity tests + timing of the main configs
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -p no:cacheprovider 2>&1 | tail -3
timeout 300 python scripts/time_variants.py ${VARIANTS:-16} 2>&1 | tail -4
timeout 300 python scripts/time_c3.py 2>&1 | tail -6
timeout 300 python bench.py --config C4 --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C4', d['ms_per_step'], d['value'])"
timeout 300 python bench.py --config C5 --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C5', d['ms_per_step'], d['value'])"
