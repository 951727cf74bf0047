timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
for c in c3 c2 c1; do echo "== $c"; timeout 300 python tools/tune.py $c 20 2>&1 | tail -20; done
echo "== c4"; timeout 600 python tools/tune.py c4 3 2>&1 | tail -12
echo "== c5"; TUNE_INSTANCES=1024 timeout 600 python tools/tune.py c5 5 2>&1 | tail -12
