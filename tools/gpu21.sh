for L in base nobar nosts; do echo "== $L"; EMPC_LIB=tools/libexp_$L.so EMPC_PHASES=1 TUNE_VARIANTS=7 TUNE_CPS=1 timeout 300 python tools/tune.py c3 10 2>&1 | grep -E "phases" | tail -1; done
