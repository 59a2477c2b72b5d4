O=gpurun_out/c65; mkdir -p $O
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_generate_gpu.py tests/test_oracle_parity_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt | cut -c1-300
for i in 1 2; do timeout 300 python bench.py --no-ft --no-cpu > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/b.json')); print(round(d['value']), d['decode_step']['ms_per_token'], [(s['n_cols'], round(s['frac'],3)) for s in d['batch_sweep']])"; done
