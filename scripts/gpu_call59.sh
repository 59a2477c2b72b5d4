O=gpurun_out/c59; mkdir -p $O
timeout 1200 python -m pytest tests/test_finetune_gpu.py tests/test_finetune_dp_gpu.py tests/test_fused_gpu.py tests/test_qlinear_gpu.py tests/test_container_gpu.py tests/test_bench_multirank_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-400
timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1
