O=gpurun_out/c22; mkdir -p $O
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]])
P
}
for V in 0 5 7; do QEFT_GEMV2_VAR=$V timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/b$V.json 2>$O/b$V.err; echo VAR=$V; summ $O/b$V.json; tail -1 $O/b$V.err; done
QEFT_GEMV2_VAR=7 timeout 300 python scripts/debug_gemv2.py > $O/dbg7.txt 2>&1; tail -4 $O/dbg7.txt
