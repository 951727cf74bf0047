timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -2
EMPC_PHASES=1 TUNE_VARIANTS=0,6,7,8,11 TUNE_CPS=1 timeout 300 python tools/tune.py c3 20 2>&1 | grep -E "phases|variant" | tail -10
TUNE_CPS=1 timeout 300 python tools/tune.py c2 20 2>&1 | grep -E "variant" | tail -10
