timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 -x 2>&1 | tail -4
EMPC_PHASES=1 TUNE_VARIANTS=-1 timeout 120 python tools/tune.py c3 20 2>&1 | grep -E "phases|persist|variant" | tail -3
for c in c3 c5; do st=30; [ $c = c5 ] && st=3; timeout 600 python bench.py --config $c --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c rollout', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['latency_ms_median'],4), 'frac', round(d['roofline']['frac'],3))"
timeout 600 python bench.py --config $c --scorer condensed --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c condensed', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['latency_ms_median'],4), 'frac', round(d['roofline']['frac'],3))"
done
