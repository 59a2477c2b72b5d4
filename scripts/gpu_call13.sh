O=gpurun_out/c13; mkdir -p $O
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in (d.get("batch_sweep") or [])], round(d["e2e"]["value"]))
P
}
for V in 4 3; do QEFT_GEMV2_VAR=$V timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_v$V.json 2>$O/bench_v$V.err; echo VAR=$V; summ $O/bench_v$V.json; done
QEFT_GEMV2_VAR=4 timeout 300 python scripts/trace_gemv.py > $O/trace_v4.txt 2>&1; cat $O/trace_v4.txt | cut -c1-250
