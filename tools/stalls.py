"""Warp-stall breakdown (all samples) from an `ncu --page source --csv` dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
ie = h.index('Instructions Executed')
tot = {c: 0 for c in cols}
for r in rows[2:]:
    try:
        int(r[ie])
    except (ValueError, IndexError):
        continue
    for c in cols:
        try:
            tot[c] += int(r[h.index(c)] or 0)
        except ValueError:
            pass
T = sum(tot.values()) or 1
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    print(f"{c:28s} {v / T:.3f}")
