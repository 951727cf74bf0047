for env in "" "EMPC_NO_PDL=1"; do
env $env timeout 300 python bench.py --config c5 --scorer condensed --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$env', round(d['ms_per_step'],3), round(d['roofline']['rollout_ms_per_launch'],3))"
done
EMPC_PHASES=1 timeout 300 python bench.py --config c5 --scorer condensed --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep phases | tail -2
EMPC_PHASES=1 timeout 300 python bench.py --config c3 --scorer condensed --steps 2 --warmup 3 --no-cpu-baseline 2>&1 | grep phases | tail -2
