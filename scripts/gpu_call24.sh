O=gpurun_out/c24; mkdir -p $O
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; tail -2 $O/pytest_gemm.txt
for S in 0 1 -1; do QEFT_GEMM_SK=$S timeout 300 python scripts/ab_gemm.py 2>&1 | tail -1 | tee -a $O/ab.txt; done
for S in 0 -1; do QEFT_GEMM_SK=$S timeout 600 python scripts/configs_perf.py > $O/configs_sk$S.json 2>$O/configs_sk$S.err; python -c "
import json,sys; d=json.load(open('$O/configs_sk$S.json')); print('SK=$S', [(g['shape'],g['T'],round(g['fwd_tflops']),round(g['dgrad_tflops'])) for g in d['gemm_13b_3bit']])"; done
