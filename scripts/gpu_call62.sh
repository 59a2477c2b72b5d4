O=gpurun_out/c62; mkdir -p $O
timeout 1500 python -m pytest tests/test_finetune_gpu.py tests/test_finetune_dp_gpu.py tests/test_fd_gpu.py tests/test_qlinear_gpu.py tests/test_oracle_parity_gpu.py tests/test_bench_multirank_gpu.py tests/test_optim_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-400
for i in 1 2; do for W in 0 1; do QEFT_WGRAD_STREAM=$W timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1 | sed "s/^/W=$W /"; done; done
