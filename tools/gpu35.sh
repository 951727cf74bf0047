# tensor-core rollout: phase / per-step cycle breakdown at C4, C5, C3
set -x
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 2>&1 | tail -4
for c in c4 c5 c3; do
  EMPC_PHASES=1 timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --tensor-cores on > gpurun_out/tcp_${c}.json 2> gpurun_out/tcp_${c}.err
  grep -E "phases|tc step" gpurun_out/tcp_${c}.err | tail -2
  python -c "import json;d=json.load(open('gpurun_out/tcp_${c}.json'));print('$c', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'])"
done
