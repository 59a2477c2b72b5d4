O=gpurun_out/c31; mkdir -p $O
timeout 120 python scripts/trace_gemm.py 4096 4096 2048 > $O/trace.txt 2>&1; echo "trace rc=$?"; tail -3 $O/trace.txt | cut -c1-600
timeout 300 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; echo "pytest rc=$?"; tail -15 $O/pytest_gemm.txt | cut -c1-300
for C in 1 2; do QEFT_GEMM_CG=$C timeout 200 python scripts/ab_gemm.py 2>&1 | tail -1 | sed "s/^/CG=$C /"; done
