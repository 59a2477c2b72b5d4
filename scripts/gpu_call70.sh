for cfg in "0 0" "0 1" "1 1" "1 0" "0 0"; do set -- $cfg; QEFT_GEMV2_PRE=$1 QEFT_GEMV2_XLDG=$2 timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/b.json')); print('PRE=$1 XLDG=$2', round(d['value']), round(d['ms_per_step'],4), [(p['launch'], round(p['us_per_launch'],2)) for p in d['roofline']['per_shape']])"; done
QEFT_GEMV2_PRE=1 QEFT_GEMV2_XLDG=1 timeout 600 python -m pytest tests/test_gemv_gpu.py -x -q 2>&1 | tail -1
