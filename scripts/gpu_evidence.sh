# The evidence committed under profiles/<round>/ (one GPU; never under torchrun):
#   tests + smoke, the default bench line, ncu launch lists, and ncu --set full captures of
#   the decode launch types and the fine-tune GEMMs. Outputs in gpurun_out/evidence/.
# usage: /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash scripts/gpu_evidence.sh'
set -x
O=gpurun_out/evidence
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -2 $O/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; tail -2 $O/smoke.txt
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 python scripts/configs_perf.py > $O/configs_perf.json 2> $O/configs_perf.err
timeout 300 python scripts/ab_gemm.py > $O/ab_gemm.txt 2>&1
timeout 300 python scripts/ab_gemm_cold.py > $O/ab_gemm_cold.txt 2>&1
timeout 600 python scripts/ft_step.py --steps 5 > $O/ft_step.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
timeout 600 ncu --metrics $M --clock-control none -k regex:gemv -c 256 --csv --log-file $O/decode_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-ft --no-dstep --no-sweep --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics $M --clock-control none --csv --log-file $O/ft_launches.csv \
  python scripts/ft_step.py --blocks 2 --steps 1 > /dev/null 2>&1
for t in qkv o gate_up down; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv2_kernel -s 2 -c 1 -o /tmp/gemv_$t \
    python scripts/prof_decode.py $t > /dev/null 2>&1
  ncu -i /tmp/gemv_$t.ncu-rep --page raw --csv > $O/gemv_${t}_raw.csv
  ncu -i /tmp/gemv_$t.ncu-rep --page source --csv > $O/gemv_${t}_source.csv
done
for c in "fwd 2" "dgrad 3"; do
  set -- $c
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s $2 -c 1 -o /tmp/g_$1 \
    python scripts/prof_gemm.py 4096x4096 > /dev/null 2>&1
  ncu -i /tmp/g_$1.ncu-rep --page raw --csv > $O/gemm_$1_4096x4096_T2048_raw.csv
done
timeout 600 ncu --set full --clock-control none -k regex:wgrad_kernel -s 1 -c 1 -o /tmp/wg python scripts/prof_gemm.py 4096x4096 > /dev/null 2>&1
ncu -i /tmp/wg.ncu-rep --page raw --csv > $O/wgrad_4096_T2048_raw.csv
ls -la $O
