python tools/e2e_breakdown.py c3; python tools/e2e_breakdown.py c1
for c in c1 c2 c3; do timeout 300 python bench.py --config $c --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), 'e2e', {k:round(v,4) for k,v in d['e2e'].items() if 'latency' in k})"; done
timeout 1200 python -m pytest tests -q -m gpu --timeout 600 2>&1 | tail -2
