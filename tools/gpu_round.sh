# Round measurement: tests, bench lines for every config, reference arm, ncu evidence.
set -x
./tools/tf32_peak > gpurun_out/tf32_peak.json
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -3 gpurun_out/bench_c3.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref.err
for c in c1 c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --cpu-sample-s 20 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --tensor-cores off > gpurun_out/bench_c4_ffma.json 2> gpurun_out/bench_c4_ffma.err
timeout 1200 python bench.py --config c5 --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; tail -2 gpurun_out/bench_c5.err
timeout 1200 python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --tensor-cores off > gpurun_out/bench_c5_ffma.json 2> gpurun_out/bench_c5_ffma.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/plain_b2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"persist|rollout" -s 4 -c 1 -o gpurun_out/prof_c3_bench python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c4.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c4.csv python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c4 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc4.log 2>&1
python bench.py --config c5 --instances 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_c5.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c5 python bench.py --config c5 --instances 1024 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_tc5.log 2>&1
tail -2 gpurun_out/ncu_f.log gpurun_out/ncu_tc4.log gpurun_out/ncu_tc5.log
