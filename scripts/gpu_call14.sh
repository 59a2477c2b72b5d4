O=gpurun_out/c14; mkdir -p $O
timeout 300 python scripts/trace_gemv.py --graph > $O/trace_g.txt 2>&1; cat $O/trace_g.txt | cut -c1-250
QEFT_GEMV2_VAR=4 timeout 300 python scripts/trace_gemv.py --graph > $O/trace_g4.txt 2>&1; cat $O/trace_g4.txt | cut -c1-250
