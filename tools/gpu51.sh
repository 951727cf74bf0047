# Dead E-column stores skipped in the tensor-core rollout: parity and C4 / C5 timing.
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 2>&1 | tail -1
for c in c4 c5; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err || tail -5 gpurun_out/t.err
  python -c "import json;d=json.load(open('gpurun_out/t.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['e2e']['latency_ms_median'], d['clocks']['sm_mhz'])"
done
