# N-split tensor-core rollout: parity, C4 timing with and without the split, C5 full-size traffic.
timeout 600 python -m pytest tests/test_gpu_tc.py -q -x --timeout 300 2>&1 | tail -3
for e in "" "EMPC_TC_NO_NSPLIT=1"; do
  env $e timeout 600 python bench.py --config c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t4.json 2> gpurun_out/t4.err || tail -5 gpurun_out/t4.err
  python -c "import json;d=json.load(open('gpurun_out/t4.json'));print('c4 [$e]', d['ms_per_step'], d['roofline']['rollout_ms_per_launch'], d['e2e']['latency_ms_median'])"
done
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -2
python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c5full python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc5.log 2>&1; tail -n 2 gpurun_out/ncu_tc5.log
