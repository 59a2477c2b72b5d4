O=gpurun_out/c53; mkdir -p $O
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_oracle_parity_gpu.py tests/test_configs_gpu.py tests/test_qlinear_gpu.py tests/test_generate_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest.txt | cut -c1-200
timeout 600 python bench.py --no-ft --no-dstep --no-cpu > $O/b.json 2>$O/b.err; python -c "
import json; d=json.load(open('$O/b.json')); print(round(d['value']), [(l['layout'], round(l['gemv_frac'],3), round(l['gemv_us'],2), round(l['gemm_fwd_tflops']), round(l['gemm_dgrad_tflops'])) for l in d['layouts']], [(s['n_cols'], round(s['frac'],3)) for s in d['batch_sweep']])"
