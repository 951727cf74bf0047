EMPC_PHASES=1 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "timeline" | tail -1
python tools/sweep.py c3 '' ''
for G in 2 3; do timeout 120 python tools/dbg_ws.py $G | tail -1; done
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -1
