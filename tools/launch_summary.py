"""Per-kernel totals and shares from an `ncu --metrics gpu__time_duration.sum --csv` launch list."""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
h = rows[hi]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split('(')[0].split('::')[-1]
    v = float(r[vi].replace(',', ''))
    scale = {'ns': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'msecond': 1.0, 'ms': 1.0, 'nsecond': 1e-6}.get(r[ui], 1.0)
    tot[name] += v * scale
    cnt[name] += 1
T = sum(tot.values())
print("%-28s %6s %12s %12s %7s" % ("kernel", "n", "total ms", "ms/matvec", "share"))
for k in sorted(tot, key=lambda k: -tot[k]):
    print("%-28s %6d %12.3f %12.3f %7.3f" % (k[:28], cnt[k], tot[k], tot[k] / reps, tot[k] / T))
