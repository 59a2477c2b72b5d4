for D in 0 2 3; do QEFT_GEMM_DIAG=$D timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | sed "s/^/DIAG=$D /"; done
QEFT_GEMM_SK=1 timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | sed "s/^/SK=1 /"
timeout 120 python scripts/trace_gemm.py 11008 4096 2048 | sed "s/^/gate /"
