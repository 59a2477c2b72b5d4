O=gpurun_out/c36; mkdir -p $O
timeout 600 python -m pytest tests/test_gemm_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gemm.txt | cut -c1-300
timeout 200 python scripts/ab_gemm.py 2>&1 | tail -1
timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1
