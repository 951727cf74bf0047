for c in "c4" "c4 --num-sims 2944"; do
  EMPC_PHASES=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/t.json 2> gpurun_out/t.err
  grep "tc step" gpurun_out/t.err | tail -1
  python -c "import json;d=json.load(open('gpurun_out/t.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'])"
done
