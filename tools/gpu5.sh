python tools/prof_solve.py c3 2 > gpurun_out/plain_c3b.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rollout -s 14 -c 1 -o gpurun_out/prof_c3_rollout2 python tools/prof_solve.py c3 2 > gpurun_out/ncu_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:select -s 10 -c 1 -o gpurun_out/prof_c3_select2 python tools/prof_solve.py c3 2 >> gpurun_out/ncu_c3.log 2>&1
tail -3 gpurun_out/ncu_c3.log
