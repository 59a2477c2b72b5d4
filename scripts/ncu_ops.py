"""Opcode histogram (weighted by executions) from an ncu source-page CSV."""
import csv, re, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
his = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
hi = his[0]; h = rows[hi]; ei = h.index('Instructions Executed'); so = h.index('Source')
cnt = collections.Counter(); tot = 0
for r in rows[hi + 1:]:
    if not r or r[0] in ('Kernel Name', 'Address'): break
    try: n = int(r[ei])
    except: continue
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z0-9_]+)', r[so].strip())
    cnt[m.group(2) if m else r[so]] += n; tot += n
print('total', tot, 'per unit', round(tot / units, 1))
for op, n in cnt.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 20):
    print(f'  {op:12s} {n:10d} {n / units:.1f}')
