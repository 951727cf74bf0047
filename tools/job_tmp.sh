python tools/sweep.py c2 '' ''
python tools/sweep.py c3 ''
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -2
