O=gpurun_out/c16; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; tail -15 $O/pytest_gpu.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; tail -3 $O/bench.err
python - <<'P'
import json
d=json.load(open("gpurun_out/c16/bench.json"))
print(round(d["value"]), round(d["ms_per_step"],3), d["roofline"]["frac"], [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in (d.get("batch_sweep") or [])], d["e2e"])
ft=d.get("finetune",{}); print("ft", ft.get("value"), ft.get("ms_per_step"), ft.get("mfu"), ft.get("dtype"), ft.get("e2e"), (ft.get("roofline") or {}).get("frac"))
print("dstep", d.get("decode_step",{}).get("ms_per_token"), "cpu", d.get("cpu_baseline"))
P
