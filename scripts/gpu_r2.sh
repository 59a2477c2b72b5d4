timeout 600 python -m pytest tests/test_gemv_gpu.py -q -x 2>&1 | tail -15
NS=1,4,16 RBWS=0,1,2,4 SMEMS=0,32768,98304 timeout 900 python scripts/gemv_sweep.py 2>&1 | tail -100
