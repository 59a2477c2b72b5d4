O=gpurun_out/c35; mkdir -p $O
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_qlinear_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gemm.txt | cut -c1-300
for X in 0 1; do for C in 1 2; do QEFT_GEMM_TMA_OUT=$X QEFT_GEMM_CG=$C timeout 200 python scripts/ab_gemm.py 2>&1 | tail -1 | sed "s/^/TMAOUT=$X CG=$C /"; done; done
for C in 1 2; do QEFT_GEMM_CG=$C timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('CG$C', 'kernel', d['kernel_us'], 'main', d['mainloop_us'], 'epi', d['epilogue_us'])"; done
