"""Top instructions of an ncu report's SASS source page by stall samples,
with the dominant stall columns (usage: ncu_hot.py report.ncu-rep [N])."""
import csv
import io
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") or "Stall" in h and i != si]
data = []
for r in rows[1:]:
    try:
        data.append((int(r[si]), r))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print(f"total samples {tot}; columns: {[hdr[i] for i in stall_cols][:3]}")
# per-column totals of the named stall reasons, when present
named = [i for i, h in enumerate(hdr) if h.lower().startswith("warp stall sampling (all samples)") is False
         and ("(All Samples)" in h and h != hdr[si])]
for n, r in sorted(data, key=lambda d: -d[0])[:top]:
    extra = []
    for i in named:
        try:
            v = int(r[i])
        except ValueError:
            continue
        if v > 0.15 * n:
            extra.append(f"{hdr[i].split(' (')[0]}={v}")
    print(f"{n:6d} {100.0 * n / tot:5.1f}%  {r[0][-5:]}  {r[1].strip()[:60]:60s} {' '.join(extra)}")
