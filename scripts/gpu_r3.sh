timeout 600 python -m pytest tests/test_gemv_gpu.py -q -x 2>&1 | tail -5
NS=1,16 RBWS=0 SMEMS=0 timeout 300 python scripts/gemv_sweep.py 2>&1 | tail -40
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 4 -c 2 -o gpurun_out/gemv_v8 python scripts/prof_gemv.py 4096x4096,11008x4096 1 > gpurun_out/ncu_v3.log 2>&1; tail -1 gpurun_out/ncu_v3.log
