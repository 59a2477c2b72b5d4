python scripts/debug_gemv.py 2>&1 | tail -16 | cut -c1-80
timeout 900 python -m pytest tests -m gpu -q 2>&1 | grep -E "passed|failed|Error|assert |^E  " | head -20
python scripts/micro_gemv.py 2>&1 | tail -16
