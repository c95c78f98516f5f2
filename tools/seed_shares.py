"""Average time and DRAM bytes per launch of each kernel in an ncu launch-list CSV."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
h, data = rows[i], rows[i + 1:]
kn, mn, mv = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value')
agg = defaultdict(lambda: defaultdict(list))
for r in data:
    if len(r) > mv:
        agg[r[kn].split('(')[0]][r[mn]].append(float(r[mv].replace(',', '')))
for k, m in agg.items():
    t = m['gpu__time_duration.sum']
    rd = sum(m['dram__bytes_read.sum']) / len(t)
    wr = sum(m['dram__bytes_write.sum']) / len(t)
    us = sum(t) / len(t) / 1e3
    print(f"{k:28s} n={len(t):3d} {us:9.1f} us  read {rd / 1e6:9.2f} MB  write {wr / 1e6:8.2f} MB  {(rd + wr) / (us * 1e3):7.1f} GB/s")
