O=gpurun_out/c37; mkdir -p $O
timeout 1500 python -m pytest tests/ -x -q -m gpu > $O/pytest_gpu.txt 2>&1; echo "pytest rc=$?"; tail -3 $O/pytest_gpu.txt | cut -c1-300
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?"; python - $O/bench.json <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["frac_of_peak"],3), "e2e", round(d["e2e"]["value"]), "ft", round(d["finetune"]["value"]), d["finetune"].get("mfu"), "dstep", d["decode_step"].get("ms_per_token"), [(s["n_cols"], round(s["frac"],3)) for s in d["batch_sweep"]])
print(json.dumps(d["roofline"])[:600])
P
