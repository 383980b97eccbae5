"""Sum the per-kernel ncu metrics of scripts/gpu_traffic.sh's captures into
profiles/r2_traffic.json: {config: {dram_bytes, ms, kernels: [...]}}."""
import csv
import json
import os
import sys

src, dst = sys.argv[1], sys.argv[2]
out = {}
for cfg in ("C2", "C3", "C3_real", "C4", "C4_real", "C5"):
    path = os.path.join(src, f"traffic_{cfg}.csv")
    if not os.path.exists(path):
        continue
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    if not rows:
        continue
    hdr = rows[0]
    ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), \
        hdr.index("Metric Unit")
    idi = hdr.index("ID")
    kern = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-6, "us": 1e-3, "usecond": 1e-3,
             "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    for r in rows[1:]:
        k = kern.setdefault(r[idi], {"kernel": r[ki][:120]})
        v = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
        k[r[mi]] = v
    ks = list(kern.values())
    total = sum(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0) for k in ks)
    ms = sum(k.get("gpu__time_duration.sum", 0) for k in ks)
    out[cfg] = {"dram_bytes": total, "ms_serialised": round(ms, 4), "launches": len(ks),
                "kernels": [{"kernel": k["kernel"], "dram_bytes": k.get("dram__bytes_read.sum", 0)
                             + k.get("dram__bytes_write.sum", 0), "ms": round(k.get("gpu__time_duration.sum", 0), 4)}
                            for k in ks]}
if "C2" in out:
    out["C2_fwd_kernel"] = dict(out["C2"])
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps({k: (v["dram_bytes"], v["ms_serialised"], v["launches"]) for k, v in out.items()}))
