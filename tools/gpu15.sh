timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -2
EMPC_PHASES=1 TUNE_VARIANTS=0,2,7,11 TUNE_CPS=1 timeout 200 python tools/tune.py c3 20 2>&1 | grep -E "phases|variant" | tail -8
python tools/prof_solve.py c3 3 7 > gpurun_out/plain_c3.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 24 --csv --log-file gpurun_out/launches_c3.csv python tools/prof_solve.py c3 3 7 > /dev/null 2>&1
