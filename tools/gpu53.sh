# Half-K persistent solve: parity (new test + full GPU suite), C3 timing with and without it.
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k half_k 2>&1 | tail -3
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -1
for e in "" "EMPC_NO_HALFK=1"; do
  env $e timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/t3.json 2> gpurun_out/t3.err || tail -5 gpurun_out/t3.err
  python -c "import json;d=json.load(open('gpurun_out/t3.json'));print('c3 [$e]', d['ms_per_step'], d['e2e']['latency_ms_median'], d['config']['kernel_variant'][-40:])"
done
