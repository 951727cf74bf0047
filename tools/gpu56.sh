# C3 variant sweep with the half-K persistent kernels.
timeout 600 python tools/tune.py c3 30 > gpurun_out/tune_c3.jsonl 2>&1; cut -c1-330 gpurun_out/tune_c3.jsonl | grep -v "^$" | tail -14
