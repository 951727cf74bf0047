timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -2
EMPC_PHASES=1 TUNE_VARIANTS=7,12,13 TUNE_CPS=1,2 timeout 300 python tools/tune.py c3 20 2>&1 | grep -E "phases|variant" | tail -12
TUNE_CPS=1,2,4 timeout 300 python tools/tune.py c2 20 2>&1 | grep -E "variant" | tail -30
TUNE_CPS=1 timeout 300 python tools/tune.py c1 20 2>&1 | grep -E "variant" | tail -30
