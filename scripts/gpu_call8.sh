O=gpurun_out/c8; mkdir -p $O
timeout 900 python scripts/debug_gemv2.py > $O/debug.txt 2>&1; cat $O/debug.txt | cut -c1-100
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in (d.get("batch_sweep") or [])], round(d["e2e"]["value"]))
P
}
timeout 300 python bench.py --no-ft --no-dstep --no-cpu > $O/bench.json 2>$O/bench.err; echo DEFAULT; summ $O/bench.json
for V in 1 2 3; do QEFT_GEMV2_VAR=$V timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_v$V.json 2>$O/bench_v$V.err; echo VAR=$V; summ $O/bench_v$V.json; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio --clock-control none -k regex:gemv2 -c 4 python scripts/prof_decode.py gate_up > $O/ncu.txt 2>&1; grep -E "duration|inst_exec|issued|stalled" $O/ncu.txt | tail -4
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
