# Variant sweep (parity vs the oracle + device solve time per compiled variant) at the full C5 size and at C4.
TUNE_INSTANCES=8192 timeout 900 python tools/tune.py c5 5 > gpurun_out/tune_c5.jsonl 2>&1
timeout 600 python tools/tune.py c4 5 > gpurun_out/tune_c4.jsonl 2>&1
tail -n 2 gpurun_out/tune_c5.jsonl gpurun_out/tune_c4.jsonl | cut -c1-200
