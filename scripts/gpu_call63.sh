O=gpurun_out/c63; mkdir -p $O
timeout 1500 python -m pytest tests/test_gemm_gpu.py tests/test_finetune_gpu.py tests/test_finetune_dp_gpu.py tests/test_fd_gpu.py tests/test_qlinear_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-400
for i in 1 2; do timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1; done
