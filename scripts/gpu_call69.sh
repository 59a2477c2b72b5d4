O=gpurun_out/c69; mkdir -p $O
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_generate_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-400
for i in 1 2; do timeout 600 python bench.py --no-ft --no-cpu --no-sweep > /tmp/b.json 2>/dev/null; python -c "
import json; d=json.load(open('/tmp/b.json')); print(round(d['value']), d['decode_step']['ms_per_token'])"; done
