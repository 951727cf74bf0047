# round measurement with the tensor-core rollout: peak, tests, benches, ncu
./tools/tf32_peak > gpurun_out/tf32_peak.json; cat gpurun_out/tf32_peak.json
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -2
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --cpu-sample-s 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c4 c5; do python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['ms_per_step'], d['e2e']['latency_ms_median'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['fp32_equivalent'])"; done
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc4.log 2>&1
python bench.py --config c5 --instances 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c5 python bench.py --config c5 --instances 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc5.log 2>&1
tail -1 gpurun_out/ncu_tc5.log
