"""Per-source-line stall samples of an ncu report (cuda,sass source page):
usage ncu_lines.py report.ncu-rep [N]"""
import collections
import csv
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.Counter()
src = {}
fname = None
cur = None
si = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        si = r.index("Warp Stall Sampling (All Samples)")
        continue
    if si is None or len(r) <= si:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
    elif cur is not None:
        try:
            agg[cur] += int(r[si])
        except ValueError:
            pass
tot = sum(agg.values())
print("total", tot)
for k, v in agg.most_common(top):
    print(f"{v:6d} {100.0 * v / tot:5.1f}%  {k[0]}:{k[1]}  {src[k]}")
