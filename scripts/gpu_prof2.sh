set -x
mkdir -p gpurun_out/prof2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|wgrad_kernel" -s 3 -c 3 -o /tmp/gemm python scripts/prof_gemm.py 11008x4096 2048 > /dev/null 2>&1
ncu -i /tmp/gemm.ncu-rep --page raw --csv > gpurun_out/prof2/gemm_11008x4096_raw.csv
ncu -i /tmp/gemm.ncu-rep --page source --csv > gpurun_out/prof2/gemm_11008x4096_source.csv
timeout 900 python bench.py > gpurun_out/prof2/bench.json 2> gpurun_out/prof2/bench.err
tail -c 300 gpurun_out/prof2/bench.json
