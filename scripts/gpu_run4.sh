python scripts/debug_gemv.py 2>&1 | tail -16
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | grep -E "passed|failed|Error|assert|^E " | head -20
python scripts/micro_gemv.py 2>&1 | tail -16
echo "--- no pdl"
QEFT_NO_PDL=1 python scripts/micro_gemv.py 2>&1 | head -5
