for D in 0 6 7; do QEFT_GEMM_DIAG=$D QEFT_GEMM_CG=1 timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('DIAG=$D', 'kernel', d['kernel_us'], 'main', d['mainloop_us'], 'epi', d['epilogue_us'], 'tfull0', d['tfull0'], 'mma_last', d['mma_last'])"; done
