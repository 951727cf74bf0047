EMPC_PHASES=1 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "timeline" | tail -1
python tools/sweep.py c3 '' ''
python tools/sweep.py c2 ''
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -1
