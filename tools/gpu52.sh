# Round measurement after the dead-store change: GPU tests, smoke, bench lines C3-C5 + reference arm, ncu of the C4 TC launch.
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -1 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --cpu-sample-s 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
for c in c3 c4 c5; do python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['ms_per_step'], d['e2e']['latency_ms_median'], d['roofline']['frac'], d['clocks'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc4.log 2>&1
ncu --set full --clock-control none -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c5full python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc5.log 2>&1
tail -n 1 gpurun_out/ncu_tc4.log gpurun_out/ncu_tc5.log
