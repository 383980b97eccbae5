"""Per-source-line executed warp instructions of an ncu report (top N)."""
import collections
import csv
import subprocess
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = collections.Counter()
src = {}
fname = cur = None
ii = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        ii = r.index("Instructions Executed")
        continue
    if ii is None or len(r) <= ii:
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
    elif cur is not None:
        try:
            agg[cur] += int(r[ii])
        except ValueError:
            pass
tot = sum(agg.values())
print("total", tot)
for k, v in agg.most_common(top):
    print(f"{v:10d} {100.0 * v / tot:5.1f}%  {k[0]}:{k[1]}  {src[k]}")
