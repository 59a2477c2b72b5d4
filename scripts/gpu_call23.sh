O=gpurun_out/c23; mkdir -p $O
timeout 900 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; tail -3 $O/pytest_gemm.txt
for S in 0 -1; do QEFT_GEMM_SK=$S timeout 300 python scripts/ab_gemm.py 2>&1 | tail -1; done
for S in 0 -1; do QEFT_GEMM_SK=$S timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1; done
