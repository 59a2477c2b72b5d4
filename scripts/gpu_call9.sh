O=gpurun_out/c9; mkdir -p $O
timeout 300 python scripts/debug_kpop.py > $O/kpop.txt 2>&1; cat $O/kpop.txt
QEFT_GEMV_V1=1 timeout 300 python scripts/debug_kpop.py > $O/kpop_v1.txt 2>&1; cat $O/kpop_v1.txt
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in (d.get("batch_sweep") or [])], round(d["e2e"]["value"]))
P
}
for V in 0 4 5; do QEFT_GEMV2_VAR=$V timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_v$V.json 2>$O/bench_v$V.err; echo VAR=$V; summ $O/bench_v$V.json; done
