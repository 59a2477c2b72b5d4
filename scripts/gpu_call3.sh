O=gpurun_out/c3; mkdir -p $O
timeout 1500 python scripts/debug_gemv2.py > $O/debug.txt 2>&1; cat $O/debug.txt
timeout 300 compute-sanitizer --tool memcheck python scripts/debug_gemv2.py one 512 1024 128 4 128 1 2 > $O/sanit.txt 2>&1; tail -30 $O/sanit.txt
