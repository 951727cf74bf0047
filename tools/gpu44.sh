timeout 300 python -m pytest tests/test_gpu_tc.py -q -x 2>&1 | tail -1
for c in "c4" "c4 --num-sims 2944" "c4 --num-sims 2944 --tensor-cores off" "c4 --num-sims 4864" "c4 --num-sims 4864 --tensor-cores off" "c3 --tensor-cores on" "c5"; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err
  python -c "import json;d=json.load(open('gpurun_out/t.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'][:90])"
done
