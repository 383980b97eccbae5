"""Aggregate an ncu --csv launch list: per kernel count, avg time, avg DRAM bytes."""
import collections
import csv
import sys

lines = open(sys.argv[1]).read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
hdr = rows[0]
iK, iM, iV, iID = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value'), hdr.index('ID')
d = collections.OrderedDict()
for r in rows[1:]:
    if len(r) <= iV:
        continue
    d.setdefault(r[iID], {'k': r[iK].split('(')[0].replace('void b200fft::', '')})[r[iM]] = r[iV]
agg = collections.OrderedDict()
for v in d.values():
    a = agg.setdefault(v['k'], [0, 0.0, 0.0])
    a[0] += 1
    a[1] += float(v.get('gpu__time_duration.sum', '0').replace(',', ''))
    a[2] += float(v.get('dram__bytes_read.sum', '0').replace(',', '')) + float(v.get('dram__bytes_write.sum', '0').replace(',', ''))
for k, (n, t, b) in agg.items():
    print(f"  {n:3d}x {k[:64]:64s} avg {t / n / 1e3:9.2f} us  avg dram {b / n / 1e6:8.1f} MB")
