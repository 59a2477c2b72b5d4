O=gpurun_out/c52; mkdir -p $O
timeout 600 python bench.py --no-ft --no-dstep --no-cpu > $O/b.json 2>$O/b.err; python -c "
import json; d=json.load(open('$O/b.json')); print([(l['layout'], round(l['gemv_frac'],3), round(l['gemm_fwd_tflops']), round(l['gemm_dgrad_tflops'])) for l in d['layouts']])"
QEFT_GEMM_SCATTER_EPI=1 timeout 600 python bench.py --no-ft --no-dstep --no-cpu > $O/b0.json 2>$O/b0.err; python -c "
import json; d=json.load(open('$O/b0.json')); print('old scatter epi', [(l['layout'], round(l['gemv_frac'],3), round(l['gemm_fwd_tflops']), round(l['gemm_dgrad_tflops'])) for l in d['layouts']])"
