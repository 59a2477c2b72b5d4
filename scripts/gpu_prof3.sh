mkdir -p gpurun_out/prof3
for L in qkv o gate_up down; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv_kernel -s 2 -c 1 -o /tmp/gemv_$L python scripts/prof_decode.py $L > /dev/null 2>&1
ncu -i /tmp/gemv_$L.ncu-rep --page raw --csv > gpurun_out/prof3/gemv_${L}_raw.csv
ncu -i /tmp/gemv_$L.ncu-rep --page source --csv > gpurun_out/prof3/gemv_${L}_source.csv
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:gemv_kernel -c 200 --csv --log-file gpurun_out/prof3/decode_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-ft > /dev/null 2>&1
timeout 900 python bench.py > gpurun_out/prof3/bench.json 2> gpurun_out/prof3/bench.err
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
ls gpurun_out/prof3
