"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel+grid."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, gi = h.index('Kernel Name'), h.index('Metric Value'), h.index('Grid Size')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    name = r[ki].split('(')[0].replace('void ', '')[:48] + ' ' + r[gi]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
print(f"total {tot / 1e3:.1f} us over {sum(v[0] for v in agg.values())} launches")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{k:70s} {v[0]:5d} {v[1] / 1e3:9.1f}us {v[1] / v[0] / 1e3:8.2f}us/launch {100 * v[1] / tot:5.1f}%")
