"""Summarise an `ncu --page source --csv` SASS dump: opcode mix and the hottest instructions."""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ie = h.index('Source'), h.index('Instructions Executed')
ss = h.index('Warp Stall Sampling (All Samples)')
c, tot, hot = Counter(), 0, []
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        if r and r[0] == 'Kernel Name':
            if tot:
                break
        continue
    toks = r[si].strip().split()
    op = toks[1] if toks[0].startswith('@') else toks[0]
    c[op.split('.')[0]] += n
    tot += n
    hot.append((int(r[ss] or 0), n, r[si].strip()))
print("warp instructions", tot)
for k, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(f"{k:10s} {v / tot:.3f}")
