timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_qlinear_gpu.py tests/test_finetune_gpu.py -q 2>&1 | tail -2
timeout 900 python scripts/ft_step.py --blocks 32 --steps 5 2>&1 | tail -1
timeout 600 python scripts/ft_prof.py 4 2>&1 | grep -E "gemm_kernel|wgrad|Self CUDA time" | cut -c1-60,180-215
