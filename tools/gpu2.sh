timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -15
for c in c3 c1 c2; do timeout 300 python bench.py --config $c --steps 50 --warmup 5 --cpu-sample-s 5 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c rc=$?"; tail -2 gpurun_out/bench_$c.err; done
timeout 600 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "c4 rc=$?"; tail -2 gpurun_out/bench_c4.err
