O=gpurun_out/c67; mkdir -p $O
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gemv_gpu.py -x -q -k "fused or swiglu" > $O/racecheck_gemv.txt 2>&1; echo "rc=$?"; tail -4 $O/racecheck_gemv.txt | cut -c1-300
timeout 1500 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_gemm_gpu.py -x -q -k "streamk_matches_whole_tiles and 512" > $O/racecheck_gemm.txt 2>&1; echo "rc=$?"; tail -4 $O/racecheck_gemm.txt | cut -c1-300
