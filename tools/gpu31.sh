timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -3
timeout 600 python tools/plant_bench.py > gpurun_out/plant_bench.json 2>&1; cat gpurun_out/plant_bench.json
timeout 300 python tools/closedloop_bench.py --periods 200 > gpurun_out/cl_single.json 2>&1; cat gpurun_out/cl_single.json
