set -x
python bench.py --config c3 --scorer condensed --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cond_ -s 8 -c 4 -o gpurun_out/prof_cond_c3 python bench.py --config c3 --scorer condensed --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cond3.log 2>&1
tail -3 gpurun_out/ncu_cond3.log
ncu --set full --clock-control none --import-source on -k regex:cond_score -s 3 -c 1 -o gpurun_out/prof_cond_c5 python bench.py --config c5 --scorer condensed --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_cond5.log 2>&1
tail -3 gpurun_out/ncu_cond5.log
