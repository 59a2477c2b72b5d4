O=gpurun_out/c6; mkdir -p $O
timeout 900 python scripts/debug_gemv2.py > $O/debug.txt 2>&1; cat $O/debug.txt | cut -c1-100
summ() { python - "$1" <<'P'
import json,sys
d=json.load(open(sys.argv[1]))
print(round(d["value"]), round(d["ms_per_step"],3), round(d["roofline"]["frac"],3), [(p["launch"], round(p["us_per_launch"],2), round(p["frac"],3)) for p in d["roofline"]["per_shape"]], [(b["n_cols"], round(b["frac"],3)) for b in d.get("batch_sweep",[])], round(d["e2e"]["value"]))
P
}
timeout 300 python bench.py --no-ft --no-dstep --no-cpu > $O/bench_gemv.json 2> $O/bench_gemv.err; tail -3 $O/bench_gemv.err; summ $O/bench_gemv.json
for S in 1 2 4; do QEFT_GEMV2_S=$S timeout 300 python bench.py --no-ft --no-dstep --no-cpu --no-sweep > $O/bench_s$S.json 2>/dev/null; echo S=$S; summ $O/bench_s$S.json; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:gemv2 -c 8 python scripts/prof_decode.py gate_up > $O/ncu_gu.txt 2>&1; grep -E "gemv2|duration|inst_exec|dram|issued|stalled" $O/ncu_gu.txt | tail -9
