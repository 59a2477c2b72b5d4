timeout 300 python scripts/ab_gemm_cold.py _ab_old | tail -1
timeout 300 python scripts/ab_gemm_cold.py | tail -1
QEFT_GEMM_TMA_OUT=0 timeout 300 python scripts/ab_gemm_cold.py | tail -1 | sed 's/^/TMAOUT0 /'
QEFT_GEMM_SK=0 timeout 300 python scripts/ab_gemm_cold.py | tail -1 | sed 's/^/SK0 /'
