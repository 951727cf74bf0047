for v in 12 13 14; do
  timeout 600 python bench.py --config c5 --steps 5 --warmup 3 --no-cpu-baseline --variant $v > gpurun_out/tcv_$v.json 2> gpurun_out/tcv_$v.err
  python -c "import json;d=json.load(open('gpurun_out/tcv_$v.json'));print('$v', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'][:60])"
done
