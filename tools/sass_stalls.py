"""Per-region stall breakdown of one kernel from an ncu SASS source export:
   ncu -i X.ncu-rep --page source --csv --print-source sass --kernel-name regex:K --launch-count 1 > f.csv
   python tools/sass_stalls.py f.csv [from to]   (instruction index range; default: top lines)"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
secs, cur = [], None
for r in rows:
    if r and r[0] == 'Kernel Name':
        cur = []; secs.append((r[1], cur)); continue
    if r and r[0] == 'Address':
        continue
    cur.append(r)
name, data = secs[0]
iS = h.index('Warp Stall Sampling (All Samples)'); iE = h.index('Instructions Executed')
cols = [c for c in h if c.startswith('stall_') and 'Not Issued' not in c]
tot = sum(float(r[iS] or 0) for r in data)
def agg(a, b):
    c = collections.Counter()
    for r in data[a:b]:
        for k in cols:
            c[k] += float(r[h.index(k)] or 0)
    return c
if len(sys.argv) > 3:
    a, b = int(sys.argv[2]), int(sys.argv[3])
    c = agg(a, b); s = sum(c.values())
    print(f'[{a},{b}) {100 * s / tot:.1f}% of samples:', ', '.join(f'{k[6:]} {100 * v / s:.0f}%' for k, v in c.most_common(6)))
else:
    c = agg(0, len(data)); s = sum(c.values())
    print(name[:60], ', '.join(f'{k[6:]} {100 * v / s:.0f}%' for k, v in c.most_common(8)))
