O=gpurun_out/c12; mkdir -p $O
timeout 300 python scripts/trace_gemv.py > $O/trace.txt 2>&1; cat $O/trace.txt | cut -c1-250
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in (d.get("batch_sweep") or [])], round(d["e2e"]["value"]))
P
}
timeout 300 python bench.py --no-ft --no-dstep --no-cpu > $O/bench.json 2>$O/bench.err; echo DEFAULT; summ $O/bench.json
for S in 1; do QEFT_GEMV2_S=$S timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_s$S.json 2>/dev/null; echo S=$S; summ $O/bench_s$S.json; done
timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.txt 2>&1; tail -5 $O/pytest_gpu.txt
