O=gpurun_out/c10; mkdir -p $O
timeout 300 python scripts/trace_gemv.py > $O/trace.txt 2>&1; cat $O/trace.txt
QEFT_GEMV2_VAR=4 timeout 300 python scripts/trace_gemv.py > $O/trace_v4.txt 2>&1; cat $O/trace_v4.txt
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
