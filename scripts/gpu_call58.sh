O=gpurun_out/c58; mkdir -p $O
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_generate_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-400
timeout 600 python bench.py --no-ft --no-cpu --no-sweep > $O/b.json 2>$O/b.err; python -c "
import json; d=json.load(open('$O/b.json')); print(round(d['value']), d['decode_step']['ms_per_token'])"
