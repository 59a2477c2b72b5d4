QEFT_GEMV_DEBUG=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o /tmp/gemv_dbg python scripts/prof_gemv.py 11008x4096 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv -s 2 -c 1 -o /tmp/gemv_v9 python scripts/prof_gemv.py 11008x4096 1 > /dev/null 2>&1
for f in gemv_dbg gemv_v9; do ncu -i /tmp/$f.ncu-rep --page raw --csv > gpurun_out/raw_$f.csv; ncu -i /tmp/$f.ncu-rep --page source --csv > gpurun_out/src_$f.csv; done
ls -la gpurun_out
