timeout 600 python bench.py --config c4 --sharded --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('c4 sharded N=1', round(d['ms_per_step'],3))"
timeout 900 python -m pytest tests -q -m gpu --timeout 600 -k "shard or radix or selection" 2>&1 | tail -2
