O=gpurun_out/c21; mkdir -p $O
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]])
P
}
for P in 2 1 0; do QEFT_GEMV2_PREX=$P timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/b$P.json 2>$O/b$P.err; echo PREX=$P; summ $O/b$P.json; done
