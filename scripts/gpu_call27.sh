O=gpurun_out/c27; mkdir -p $O
timeout 900 python -m pytest tests/test_gemv_gpu.py tests/test_oracle_parity_gpu.py -x -q > $O/pytest.txt 2>&1; tail -1 $O/pytest.txt
for C in 1 2; do QEFT_GEMV2_CONTIG=$C timeout 400 python bench.py --no-ft --no-dstep --no-cpu > $O/b$C.json 2>$O/b$C.err; python - $O/b$C.json $C <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print("CONTIG", sys.argv[2], round(d["value"]), round(d["ms_per_step"],3), [(s["n_cols"], round(s["frac"],3), round(s["ms_per_step"],3)) for s in d["batch_sweep"]])
P
done
QEFT_GEMV2_LOG=1 timeout 400 python bench.py --no-ft --no-dstep --no-cpu 2>&1 >/dev/null | grep gemv2 | sort | uniq
