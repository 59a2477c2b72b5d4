O=gpurun_out/c28; mkdir -p $O
for D in 0 2 4; do QEFT_GEMM_DIAG=$D timeout 300 python scripts/ab_gemm.py 2>&1 | tail -1 | sed "s/^/DIAG=$D /"; done
