mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu --timeout 400 -x 2>&1 | tail -3
for st in 0 150 300; do for wt in 224 352; do
EMPC_STAGGER=$st EMPC_WS_THREADS=$wt TUNE_VARIANTS=12 timeout 300 python tools/tune.py c3 30 2>&1 | python -c "import sys,json; [print('st=$st wt=$wt', round(json.loads(l)['solve_ms'],4), json.loads(l)['desc'][-60:]) for l in sys.stdin if l.startswith('{')]"
done; done
TUNE_VARIANTS=7 timeout 300 python tools/tune.py c3 30 2>&1 | python -c "import sys,json; [print('v7', round(json.loads(l)['solve_ms'],4)) for l in sys.stdin if l.startswith('{')]"
EMPC_PHASES=1 EMPC_VARIANT=12 EMPC_STAGGER=150 timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "phases|persist" | tail -2
