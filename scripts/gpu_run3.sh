python scripts/debug_gemv.py 2>&1 | tail -20
echo "---- no PDL"
QEFT_NO_PDL=1 python scripts/debug_gemv.py 2>&1 | tail -20
timeout 900 python -m pytest tests/test_gemv_gpu.py -q -x 2>&1 | grep -E "Error|assert|worst|^E " | head -30
