for G in 2 3 10; do timeout 120 python tools/dbg_ws.py $G | tail -1; done
timeout 900 python -m pytest tests -q -m gpu --timeout 300 2>&1 | tail -3
