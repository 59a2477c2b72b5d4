O=gpurun_out/c25; mkdir -p $O
for S in 0 1; do QEFT_GEMM_SK=$S ncu --clock-control none -k regex:gemm_kernel -s 3 -c 1 --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,gpc__cycles_elapsed.max,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg --csv python scripts/sk_probe.py > $O/ncu_sk$S.csv 2>&1; done
QEFT_GEMM_SK=1 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm_sk1 python scripts/sk_probe.py > /dev/null 2>&1
QEFT_GEMM_SK=0 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3 -c 1 -o $O/gemm_sk0 python scripts/sk_probe.py > /dev/null 2>&1
ls -la $O
