timeout 900 python -m pytest tests/test_gemv_gpu.py -q 2>&1 | grep -E "passed|failed|Error|assert |^E  " | head -10
python scripts/micro_gemv.py 2>&1 | head -5
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 1 -c 2 -o gpurun_out/gemv9 python scripts/prof_gemv.py 8192x28672,4096x4096 1 > gpurun_out/ncu9.log 2>&1; tail -1 gpurun_out/ncu9.log
