for dbg in 0 1 3 5 2; do echo "dbg $dbg";
QEFT_GEMV_DEBUG=$dbg NS=1 RBWS=0 SMEMS=0 timeout 300 python scripts/gemv_sweep.py 2>&1 | tail -5 | cut -c1-90 | head -3
done
