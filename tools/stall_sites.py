"""Instructions with the most samples of one stall reason (ncu --page source --csv dump)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
col = h.index(sys.argv[2])
si, ad, ie = h.index('Source'), h.index('Address'), h.index('Instructions Executed')
out, seen = [], set()
for i, r in enumerate(rows[2:]):
    try:
        v = int(r[col] or 0)
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    if r[ad] in seen:
        continue
    seen.add(r[ad])
    out.append((v, r[ad][-5:], n, r[si].strip()[:60], i))
out.sort(reverse=True)
for v, a, n, src, i in out[:int(sys.argv[3]) if len(sys.argv) > 3 else 12]:
    print(v, a, n, src)
