# Box diagnostics: memory-system microbenchmarks and the C2 ring knobs (box-to-box spread)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
nvidia-smi --query-gpu=name,serial,clocks.max.sm,clocks.max.mem,ecc.mode.current,power.limit --format=csv
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("L2", p.L2_cache_size, "SMs", p.multi_processor_count)
import ctypes
rt = ctypes.CDLL("libcudart.so") if False else None
PY
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fb scripts/fabric_bench.cu && /tmp/fb
for r in 24 40 56; do echo "ring margin $r: $(B200FFT_AB_RING=$r timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"; done
echo "no persist: $(B200FFT_AB_PERSIST=0 timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"
echo "default: $(timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"
echo "Y evict-last: $(B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=16384 timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"
