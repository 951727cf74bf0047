timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k "c2_g3" 2>&1 | grep -E "Error|error|passed|failed" | head -5
TUNE_VARIANTS=0 TUNE_CPS=1 timeout 200 python tools/tune.py c3 5 2>&1 | grep -E "variant" | tail -2
