for i in 1 2; do timeout 300 python bench.py --no-ft --no-dstep --no-cpu > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/b.json')); print(round(d['value']), [(s['n_cols'], round(s['frac'],3)) for s in d['batch_sweep']])"; done
