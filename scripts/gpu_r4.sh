timeout 600 python -m pytest tests/test_gemv_gpu.py -q -x 2>&1 | tail -3
NS=1 RBWS=0 SMEMS=0 timeout 300 python scripts/gemv_sweep.py 2>&1 | tail -5
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e'], [ (r['shape'], round(r['us_per_launch'],2), round(r['frac'],3)) for r in d['roofline']['per_shape']])"
