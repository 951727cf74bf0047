for v in 0 7; do EMPC_PHASES=1 TUNE_VARIANTS=$v TUNE_CPS=1 timeout 200 python tools/tune.py c3 10 2>&1 | grep -E "phases|variant" | tail -2; done
EMPC_PHASES=1 TUNE_VARIANTS=0 TUNE_CPS=1 timeout 200 python tools/tune.py c2 10 2>&1 | grep -E "phases|variant" | tail -2
EMPC_PHASES=1 TUNE_VARIANTS=0 TUNE_CPS=1 timeout 200 python tools/tune.py c1 10 2>&1 | grep -E "phases|variant" | tail -2
EMPC_PHASES=1 TUNE_VARIANTS=2 TUNE_CPS=0 timeout 300 python tools/tune.py c4 3 2>&1 | grep -E "phases|variant" | tail -2
