O=gpurun_out/c2; mkdir -p $O
timeout 600 python -m pytest tests/test_gemv_gpu.py tests/test_configs_gpu.py tests/test_oracle_parity_gpu.py -x -q > $O/pytest_gemv.txt 2>&1; tail -15 $O/pytest_gemv.txt
timeout 300 python bench.py --no-ft --no-dstep --no-cpu > $O/bench_gemv.json 2> $O/bench_gemv.err; tail -3 $O/bench_gemv.err
timeout 300 env QEFT_GEMV_V1=1 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_gemv_v1.json 2> $O/bench_gemv_v1.err
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
