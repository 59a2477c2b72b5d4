for S in -1 1; do QEFT_GEMM_SK=$S timeout 300 python scripts/ab_gemm_cold.py | tail -1 | sed "s/^/SK=$S /"; QEFT_GEMM_SK=$S timeout 300 python scripts/ab_gemm.py | tail -1; done
