python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
python - <<'PY'
import torch
p = torch.cuda.get_device_properties(0)
print("persisting L2 max:", torch.cuda.get_device_properties(0).L2_cache_size)
import ctypes
cudart = ctypes.CDLL("libcudart.so.12") if False else None
PY
for x in 0 2048 2 8 64 72 0; do echo "xo=$x $(B200FFT_ALLOW_WRONG=1 B200FFT_AB_XOPTS=$x timeout -s KILL 120 python scripts/time_c2.py 10 | tail -1)"; done
