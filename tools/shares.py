"""Summarise an ncu launch-list CSV (gpu__time_duration.sum per launch) by kernel."""
import csv, sys
for path in sys.argv[1:]:
    rows = list(csv.reader(open(path)))
    i = [k for k, r in enumerate(rows) if 'Kernel Name' in r][0]
    hdr, data = rows[i], rows[i + 1:]
    kn, mv, mn = hdr.index('Kernel Name'), hdr.index('Metric Value'), hdr.index('Metric Name')
    agg, tot = {}, 0.0
    for r in data:
        if len(r) <= mv or r[mn] != 'gpu__time_duration.sum':
            continue
        name = r[kn].split('(')[0]
        v = float(r[mv].replace(',', ''))
        a = agg.setdefault(name, [0.0, 0, 0.0]); a[0] += v; a[1] += 1; a[2] = max(a[2], v); tot += v
    print(f"== {path}  total {tot/1e3:.1f} us")
    for k, (v, n, mx) in sorted(agg.items(), key=lambda x: -x[1][0])[:12]:
        print(f"{k:40s} {v/1e3:10.1f}us {n:4d} max {mx/1e3:9.1f}us {100*v/tot:6.2f}%")
