timeout 200 python tools/steps.py 0 2>&1 | tail -5
DOF=6 timeout 200 python tools/steps.py 0 2>&1 | tail -5
python tools/prof_solve.py c3 2 > gpurun_out/plain_c3c.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:rollout -s 14 -c 1 -o gpurun_out/prof_c3_rollout3 python tools/prof_solve.py c3 2 > gpurun_out/ncu_c3.log 2>&1; tail -2 gpurun_out/ncu_c3.log
