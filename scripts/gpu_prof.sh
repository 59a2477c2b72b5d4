# ncu evidence for profiles/ (one GPU; never under torchrun)
set -x
mkdir -p gpurun_out/prof
# 1. launch list of the decode bench's GEMV launches (cold-cache, serialised: shares, not absolutes)
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemv_kernel -c 300 --csv --log-file gpurun_out/prof/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-ft > /dev/null 2>&1
# 2. full capture of the GEMV per 7B shape
for sh in 4096x4096 11008x4096 4096x11008; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o /tmp/gemv_$sh python scripts/prof_gemv.py $sh 1 > /dev/null 2>&1
ncu -i /tmp/gemv_$sh.ncu-rep --page raw --csv > gpurun_out/prof/gemv_${sh}_raw.csv
ncu -i /tmp/gemv_$sh.ncu-rep --page source --csv > gpurun_out/prof/gemv_${sh}_source.csv
done
# 3. full capture of the fine-tune GEMMs (fwd, dgrad, wgrad) at T=2048
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel|wgrad_kernel" -s 3 -c 3 -o /tmp/gemm python scripts/prof_gemm.py 11008x4096 2048 > /dev/null 2>&1
ncu -i /tmp/gemm.ncu-rep --page raw --csv > gpurun_out/prof/gemm_11008x4096_raw.csv
ncu -i /tmp/gemm.ncu-rep --page source --csv > gpurun_out/prof/gemm_11008x4096_source.csv
ls -la gpurun_out/prof
