# ncu of the tensor-core rollout at C4 (one launch)
python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --tensor-cores on > gpurun_out/tc_c4_plain.json 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout_tc -s 3 -c 1 -o gpurun_out/prof_tc_c4 \
  python bench.py --config c4 --steps 2 --warmup 3 --no-cpu-baseline --tensor-cores on > gpurun_out/ncu_tc_c4.log 2>&1
tail -3 gpurun_out/ncu_tc_c4.log
