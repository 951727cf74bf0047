for c in c5 c4; do
  EMPC_PHASES=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tcp_$c.json 2> gpurun_out/tcp_$c.err
  grep phases gpurun_out/tcp_$c.err | tail -1
  python -c "import json;d=json.load(open('gpurun_out/tcp_$c.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['config']['kernel_variant'][:60])"
done
