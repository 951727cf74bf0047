# tensor-core rollout: parity tests, then C4 / C5 / C3 bench with and without it
set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 2>&1 | tail -15
for c in c4 c5 c3 c2; do
  for t in on off; do
    timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --tensor-cores $t > gpurun_out/tc_${c}_$t.json 2> gpurun_out/tc_${c}_$t.err
    python -c "import json;d=json.load(open('gpurun_out/tc_${c}_$t.json'));print('$c $t', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'][:60])"
  done
done
