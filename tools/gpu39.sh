timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -2
for c in c4 c5 c3; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --tensor-cores on > gpurun_out/tc_$c.json 2> gpurun_out/tc_$c.err
  python -c "import json;d=json.load(open('gpurun_out/tc_$c.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'])"
done
