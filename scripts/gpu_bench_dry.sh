# Dry run of bench.py's N > 1 paths on one GPU (ranks share cuda:0, gloo + host collectives)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out
B200FFT_BENCH_SHARE_GPU=1 timeout -s KILL 900 python bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/dry2.json 2> gpurun_out/dry2.err; echo rc=$?
python - <<'PY'
import json
ln = [l for l in open("gpurun_out/dry2.json") if l.startswith("{")]
d = json.loads(ln[-1])
print({k: d.get(k) for k in ("n_gpus", "value", "dry_run")})
for k, v in d.get("extra", {}).get("sharded", {}).items():
    print(k, {x: v.get(x) for x in ("error", "n_gpus", "ms_per_step", "roundtrip_rel_l2", "dry_run", "gpu_launches")})
    print(k, "phases", v.get("phases_ms"))
PY
tail -5 gpurun_out/dry2.err
