# Round measurement: tests, bench lines for every config, reference arms, ncu
# evidence; everything lands in gpurun_out/r02/ (copied to profiles/ by hand).
set -x
O=gpurun_out/r02; mkdir -p $O
./tools/ffma_peak > $O/peaks.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ffma2_probe tools/ffma2_probe.cu && /tmp/ffma2_probe > $O/ffma2_probe_r02.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -o /tmp/graph_io_probe tools/graph_io_probe.cu && /tmp/graph_io_probe > $O/graph_io_probe_r02.txt 2>&1
timeout 1500 python -m pytest tests -q -m gpu --timeout 600 > $O/pytest_gpu_r02.log 2>&1; tail -2 $O/pytest_gpu_r02.log
timeout 600 python bench.py > $O/bench_c3_r02.json 2> $O/bench_c3.err
for c in c1 c2; do timeout 300 python bench.py --config $c > $O/bench_${c}_r02.json 2> $O/bench_$c.err; done
timeout 900 python bench.py --config c4 --steps 10 --warmup 3 --cpu-sample-s 20 > $O/bench_c4_r02.json 2> $O/bench_c4.err
timeout 1500 python bench.py --config c5 --steps 5 --warmup 3 --cpu-sample-s 20 > $O/bench_c5_r02.json 2> $O/bench_c5.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 2 > $O/bench_ref_c3_r02.json 2> $O/bench_ref.err
timeout 600 python bench.py --impl reference --config c5 --steps 5 --warmup 1 > $O/bench_ref_c5_r02.json 2> $O/bench_ref5.err
EMPC_PHASES=1 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "phases|persist|first sel" | tail -4 > $O/phases_c3_r02.txt
EMPC_PHASES=1 EMPC_PHASES_GEN=0 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep -E "phases|persist|first sel" | tail -4 > $O/phases_c3_gen0_r02.txt
EMPC_PHASES=1 EMPC_PHASES_GEN=0 timeout 120 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --l2 warm 2>&1 >/dev/null | grep -E "phases|persist|first sel" | tail -4 > $O/phases_c3_gen0_l2warm_r02.txt
timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --l2 warm > $O/bench_c3_l2warm_experiment_r02.json 2>/dev/null
timeout 900 python tools/closedloop_bench.py > $O/closedloop_single_r02.json 2> $O/closedloop.err
for c in c1 c2 c3 c4; do
  python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches_${c}_r02.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:persist -s 2 -c 1 -o $O/prof_c3_persist_r02 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:small -s 2 -c 1 -o $O/prof_c1_small_r02 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline > $O/ncu_c1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select_radix -s 3 -c 1 -o $O/prof_c4_radix_r02 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_c4.log 2>&1
for c in c1 c2 c3 c4 c5; do python -c "import json; d=json.load(open('$O/bench_${c}_r02.json')); print('$c', round(d['ms_per_step'],4), 'e2e med', round(d['e2e']['latency_ms_median'],4), 'mean', round(d['e2e']['latency_ms_mean'],4), 'frac', round(d['roofline']['frac'],3), d['roofline']['bound'], d['clocks'])"; done
