timeout 900 python -m pytest tests/test_qlinear_gpu.py tests/test_finetune_gpu.py -q -x -s 2>&1 | tail -30
