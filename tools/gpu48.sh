# Verify the reverted (shipped) build: C4 / C3 timing and the TC parity tests.
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 2>&1 | tail -1
for c in c4 c4 c3; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err || tail -5 gpurun_out/t.err
  python -c "import json;d=json.load(open('gpurun_out/t.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['clocks'])"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv
