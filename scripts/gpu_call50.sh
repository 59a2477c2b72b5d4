O=gpurun_out/c50; mkdir -p $O
timeout 900 python -m pytest tests/test_fused_gpu.py tests/test_finetune_gpu.py tests/test_finetune_dp_gpu.py -x -q > $O/pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest.txt | cut -c1-300
timeout 600 python _ab_old/ft_step_old.py --steps 5 2>&1 | tail -1 | sed 's/^/OLD /'
timeout 600 python scripts/ft_step.py --steps 5 2>&1 | tail -1 | sed 's/^/NEW /'
