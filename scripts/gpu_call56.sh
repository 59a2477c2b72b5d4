for V in 0 1; do QEFT_GEMV2_NT2=$V QEFT_GEMV2_LOG=1 timeout 300 python bench.py --no-ft --no-dstep --no-cpu > /tmp/b.json 2>/tmp/b.err; python -c "
import json; d=json.load(open('/tmp/b.json')); print('NT2=$V', [(s['n_cols'], round(s['frac'],3)) for s in d['batch_sweep']])"; grep "n=16" /tmp/b.err | sort | uniq; done
