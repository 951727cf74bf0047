timeout 600 python -m pytest tests/test_gpu_condensed.py -x -q -m gpu --timeout 120 2>&1 | tail -3
for c in c1 c2 c3 c4 c5; do
st=20; [ $c = c5 ] && st=3; [ $c = c4 ] && st=5
timeout 300 python bench.py --config $c --scorer condensed --steps $st --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['latency_ms_median'],4), 'launch', round(d['roofline']['rollout_ms_per_launch'],4), 'frac', round(d['roofline']['frac'],3), d['config']['kernel_variant'][:60])"
done
EMPC_PHASES=1 timeout 300 python bench.py --config c3 --scorer condensed --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep phases | tail -1
