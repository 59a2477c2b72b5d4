timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|wgrad_kernel" -s 3 -c 3 -o /tmp/gemm1 python scripts/prof_gemm.py 4096x4096 2048 > /tmp/ncu.log 2>&1; tail -2 /tmp/ncu.log
ncu -i /tmp/gemm1.ncu-rep --page raw --csv > gpurun_out/raw_gemm1.csv; ncu -i /tmp/gemm1.ncu-rep --page source --csv > gpurun_out/src_gemm1.csv
