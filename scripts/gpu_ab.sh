for v in old new old new; do QEFT_LIB_PATH=scripts/ab/lib_$v.so python scripts/ab_gemm.py; done
