O=gpurun_out/c5; mkdir -p $O
timeout 900 python scripts/debug_gemv2.py > $O/debug.txt 2>&1; cat $O/debug.txt
timeout 300 python bench.py --no-ft --no-dstep --no-cpu > $O/bench_gemv.json 2> $O/bench_gemv.err; tail -3 $O/bench_gemv.err
python - <<'P'
import json
d=json.load(open("gpurun_out/c5/bench_gemv.json"))
print(d["value"], d["ms_per_step"], d["roofline"]["frac"]); print([(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]]); print([(b["n_cols"], round(b["frac"],3)) for b in d.get("batch_sweep",[])]); print(d["e2e"])
P
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemv2_kernel -s 2 -c 1 -o /tmp/g2 python scripts/prof_decode.py gate_up > $O/ncu.log 2>&1
ncu -i /tmp/g2.ncu-rep --page raw --csv > $O/gemv2_gate_up_raw.csv 2>/dev/null
ncu -i /tmp/g2.ncu-rep --page source --csv > $O/gemv2_gate_up_source.csv 2>/dev/null
ncu -i /tmp/g2.ncu-rep --page details > $O/gemv2_gate_up_details.txt 2>/dev/null
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
