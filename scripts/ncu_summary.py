"""Summarize an ncu report exported as raw/source CSV: per-kernel key metrics,
stall reasons and the hottest SASS lines."""
import csv, sys
raw, src = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(raw)))
h = rows[0]
def f(v):
    try: return float(v)
    except: return 0.0
keys = ['Grid Size', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'sm__warps_active.avg.pct_of_peak_sustained_active',
        'sm__inst_issued.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active']
for r in rows[2:]:
    print({k: r[h.index(k)] for k in keys if k in h})
    items = [(h[i], f(r[i])) for i in range(len(h)) if 'stall' in h[i] and 'ratio' in h[i] and 'not_issued' not in h[i]]
    print('   stalls:', [(k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''), round(v, 2)) for k, v in sorted(items, key=lambda x: -x[1])[:7]])
rows = list(csv.reader(open(src)))
his = [i for i, r in enumerate(rows) if r and r[0] == 'Address']
hi = his[0]
h = rows[hi]; si = h.index('Warp Stall Sampling (All Samples)'); so = h.index('Source')
data = []
for r in rows[hi + 1:]:
    if not r or r[0] in ('Kernel Name', 'Address'): break
    try: data.append((int(r[si]), r[0][-5:], r[so]))
    except: pass
tot = sum(d[0] for d in data)
print('samples', tot)
for s, a, t in sorted(data, key=lambda x: -x[0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 15]:
    print(' ', s, round(100 * s / tot, 1), a, t.strip())
