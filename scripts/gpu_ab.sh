# A/B the GEMM builds under scripts/ab/ (usage: bash scripts/gpu_ab.sh old new [...])
libs="${@:-old new}"
for r in 1 2; do for v in $libs; do QEFT_LIB_PATH=scripts/ab/lib_$v.so python scripts/ab_gemm.py; done; done
