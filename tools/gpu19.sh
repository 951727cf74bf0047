EMPC_PHASES=1 TUNE_VARIANTS=7,12 TUNE_CPS=1 timeout 300 python tools/tune.py c3 20 2>&1 | grep -E "phases|variant" | tail -6
