O=gpurun_out/c33; mkdir -p $O
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gemm.txt | cut -c1-300
for E in 0 1; do for C in 1 2; do QEFT_GEMM_EPI=$E QEFT_GEMM_CG=$C timeout 200 python scripts/ab_gemm.py 2>&1 | tail -1 | sed "s/^/EPI=$E CG=$C /"; done; done
QEFT_GEMM_CG=1 timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('CG1', 'kernel', d['kernel_us'], 'main', d['mainloop_us'], 'epi', d['epilogue_us'])"
QEFT_GEMM_CG=2 timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('CG2', 'kernel', d['kernel_us'], 'main', d['mainloop_us'], 'epi', d['epilogue_us'])"
