for D in 0 2 3 5; do QEFT_GEMM_DIAG=$D timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('DIAG=$D', 'kernel', d['kernel_us'], 'setup', d['setup'][1], 'mma0', d['mma0'][1], 'main', d['mainloop_us'], 'epi', d['epilogue_us'])"; done
