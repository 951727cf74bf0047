timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 120 2>&1 | tail -5
echo "== c3"; TUNE_CPS=1,2,4,7 timeout 400 python tools/tune.py c3 20 2>&1 | grep -v "^$" | tail -60
echo "== c2"; TUNE_CPS=1,2,4 timeout 200 python tools/tune.py c2 20 2>&1 | tail -30
echo "== steps"; timeout 200 python tools/steps.py 2>&1 | tail -5
