# C3 measurement with the half-K persistent solve: bench line, reference arm, launch list, ncu of the persist kernel.
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python -c "import json;d=json.load(open('gpurun_out/bench_c3.json'));print('c3', d['ms_per_step'], d['e2e']['latency_ms_median'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/bench_ref_c3.json 2> gpurun_out/bench_ref.err; head -c 200 gpurun_out/bench_ref_c3.json; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"persist" -s 4 -c 1 -o gpurun_out/prof_c3_bench python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; tail -n 1 gpurun_out/ncu_f.log
