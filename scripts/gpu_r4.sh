timeout 600 python -m pytest tests/test_gemv_gpu.py tests/test_qlinear_gpu.py -q -x 2>&1 | tail -2
for dbg in 0 3 5 0; do echo "dbg $dbg";
QEFT_GEMV_DEBUG=$dbg NS=1 RBWS=0 SMEMS=0 timeout 300 python scripts/gemv_sweep.py 2>&1 | tail -5 | cut -c1-90
done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu --no-ft 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']), round(d['ms_per_step'],3), [ (r['shape'], round(r['us_per_launch'],2), round(r['frac'],3)) for r in d['roofline']['per_shape']])"
