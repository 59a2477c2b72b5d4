O=gpurun_out/c7; mkdir -p $O
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], round(d["e2e"]["value"]))
P
}
for V in 0 1 2 3; do QEFT_GEMV2_VAR=$V timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_v$V.json 2>$O/bench_v$V.err; echo VAR=$V; summ $O/bench_v$V.json; done
for V in 0 1; do QEFT_GEMV2_VAR=$V timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__warps_active.avg.per_cycle_active --clock-control none -k regex:gemv2 -c 4 python scripts/prof_decode.py gate_up > $O/ncu_v$V.txt 2>&1; grep -E "duration|inst_exec|issued|stalled|warps_active" $O/ncu_v$V.txt | tail -5; done
QEFT_GEMV2_VAR=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemv2 -s 2 -c 1 -o /tmp/v1 python scripts/prof_decode.py gate_up > /dev/null 2>&1
ncu -i /tmp/v1.ncu-rep --page source --csv > $O/v1_source.csv 2>/dev/null; ncu -i /tmp/v1.ncu-rep --page raw --csv > $O/v1_raw.csv 2>/dev/null
