"""Group the SASS of one kernel (ncu --page source --csv) by execution count: each distinct
count is (roughly) one basic block; print its share of all instructions and its opcode mix."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ie, ad = h.index('Source'), h.index('Instructions Executed'), h.index('Address')
seen, data = set(), []
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    if r[ad] in seen:
        continue
    seen.add(r[ad])
    toks = r[si].strip().split()
    op = toks[1] if toks[0].startswith('@') else toks[0]
    data.append((n, op.split('.')[0]))
tot = sum(n for n, _ in data)
lv = collections.defaultdict(collections.Counter)
for n, op in data:
    lv[n][op] += 1
print("total warp instructions", tot)
for n in sorted(lv, key=lambda n: -n * sum(lv[n].values()))[:int(sys.argv[2]) if len(sys.argv) > 2 else 10]:
    ops = lv[n]
    print("%12d x %4d  %.3f  %s" % (n, sum(ops.values()), n * sum(ops.values()) / tot, dict(ops.most_common(10))))
