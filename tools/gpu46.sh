# Round re-measurement after the container rebuild: GPU tests, every bench line, reference arm, launch lists, ncu of c3/c4.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err; cat gpurun_out/bench_c3.json | head -c 400
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref.err
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --cpu-sample-s 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 1200 python bench.py --config c5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err
for c in c1 c2 c3 c4 c5; do python -c "import json;d=json.load(open('gpurun_out/bench_$c.json'));print('$c', d['ms_per_step'], d['e2e']['value'] if isinstance(d.get('e2e'),dict) else None, d['roofline']['frac'])"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"persist" -s 4 -c 1 -o gpurun_out/prof_c3_bench python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc4.log 2>&1
tail -2 gpurun_out/ncu_f.log gpurun_out/ncu_tc4.log
