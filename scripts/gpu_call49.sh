O=gpurun_out/c49; mkdir -p $O
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_qlinear_gpu.py -x -q > $O/pytest_gemm.txt 2>&1; echo "pytest rc=$?"; tail -2 $O/pytest_gemm.txt | cut -c1-200
timeout 300 python scripts/ab_gemm_cold.py _ab_old | tail -1
timeout 300 python scripts/ab_gemm_cold.py | tail -1
timeout 600 python _ab_old/ft_step_old.py --steps 5 2>&1 | tail -1 | sed 's/^/OLD /'
timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1 | sed 's/^/NEW /'
