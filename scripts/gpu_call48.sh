timeout 600 python scripts/skinny_ab.py
QEFT_GEMM_SK=1 timeout 300 python scripts/ab_gemm_cold.py | tail -1 | sed 's/^/SK1 /'
timeout 300 python scripts/ab_gemm_cold.py | tail -1 | sed 's/^/AUTO /'
