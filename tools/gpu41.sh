for c in c5 c4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/tc_$c.json 2> gpurun_out/tc_$c.err
  python -c "import json;d=json.load(open('gpurun_out/tc_$c.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'][:50])"
done
