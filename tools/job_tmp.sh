EMPC_PHASES=1 EMPC_PHASES_GEN=5 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "phases|timeline" | tail -3
python tools/sweep.py c3 '' ''
python tools/sweep.py c2 ''
