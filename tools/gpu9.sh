timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 120 2>&1 | tail -5
echo "== c3"; TUNE_CPS=1,2 timeout 400 python tools/tune.py c3 20 2>&1 | grep -v "^$" | tail -60
echo "== c3 nopdl"; EMPC_NO_PDL=1 TUNE_VARIANTS=0,7,10,11 TUNE_CPS=1 timeout 400 python tools/tune.py c3 20 2>&1 | grep -v "^$" | tail -60
