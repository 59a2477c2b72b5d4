O=gpurun_out/c66; mkdir -p $O
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemm_gpu.py -x -q -k "streamk or pairs or wgrad_weak_multi or 300" > $O/memcheck_gemm.txt 2>&1; echo "gemm memcheck rc=$?"; tail -5 $O/memcheck_gemm.txt | cut -c1-300
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gemv_gpu.py -x -q -k "fused or swiglu or multi" > $O/memcheck_gemv.txt 2>&1; echo "gemv memcheck rc=$?"; tail -5 $O/memcheck_gemv.txt | cut -c1-300
