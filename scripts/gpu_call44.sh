for i in 1 2; do timeout 300 python scripts/ab_gemm_cold.py _ab_old | tail -1; timeout 300 python scripts/ab_gemm_cold.py | tail -1; done
