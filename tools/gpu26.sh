set -x
./tools/ffma_peak > gpurun_out/peak64.log 2>&1; cat gpurun_out/peak64.log
for c in c1 c2 c3; do timeout 300 python bench.py --config $c --scorer condensed --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/cond_$c.json 2> gpurun_out/cond_$c.err; tail -2 gpurun_out/cond_$c.err; done
timeout 300 python bench.py --config c4 --scorer condensed --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cond_c4.json 2> gpurun_out/cond_c4.err; tail -2 gpurun_out/cond_c4.err
timeout 300 python bench.py --config c5 --scorer condensed --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cond_c5.json 2> gpurun_out/cond_c5.err; tail -2 gpurun_out/cond_c5.err
for c in c1 c2 c3 c4 c5; do python -c "
import json; d=json.load(open('gpurun_out/cond_$c.json')); print('$c', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['latency_ms_median'],4), 'frac', round(d['roofline']['frac'],3), d['roofline']['achieved'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'])"; done
