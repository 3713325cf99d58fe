"""Aggregate an ncu --page source --csv dump (SASS) by opcode: stall samples and executed instructions."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hi = [k for k, r in enumerate(rows) if r and r[0] == 'Address'][0]
h = rows[hi]; data = [r for r in rows[hi + 1:] if r and r[0].startswith('0x')]
iS = h.index('Warp Stall Sampling (All Samples)'); iE = h.index('Instructions Executed'); iSrc = h.index('Source')
num = lambda v: int(v) if v and v.isdigit() else 0
tot = sum(num(r[iS]) for r in data) or 1
c, ce = Counter(), Counter()
for r in data:
    parts = r[iSrc].split()
    if not parts: continue
    op = parts[1] if parts[0].startswith('@') else parts[0]
    op = op.split('.')[0]
    c[op] += num(r[iS]); ce[op] += num(r[iE])
print('total samples', tot, 'executed', sum(ce.values()))
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} samples {v:7d} ({100*v/tot:5.1f}%) exec {ce[op]}")
