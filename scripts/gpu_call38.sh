O=gpurun_out/c38; mkdir -p $O
run() { env "$@" timeout 600 python bench.py --no-cpu --no-dstep --no-sweep > $O/b.json 2>$O/b.err; python -c "
import json; d=json.load(open('$O/b.json')); ft=d['finetune']; print('$*', round(ft['value']), round(ft['ms_per_step'],2), round(d['value']))"; }
run X=1
run QEFT_GEMM_SK=0
run QEFT_GEMM_TMA_OUT=0
run QEFT_WEAK_VIEW=0
run QEFT_GEMM_SK=0 QEFT_GEMM_TMA_OUT=0 QEFT_WEAK_VIEW=0
