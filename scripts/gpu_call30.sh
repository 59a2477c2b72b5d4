for D in 4 5; do QEFT_GEMM_DIAG=$D timeout 120 python scripts/trace_gemm.py 4096 4096 2048 | sed "s/^/DIAG=$D /"; done
