set -x
timeout 300 python -m pytest tests/test_closedloop.py -q -m gpu --timeout 200 2>&1 | tail -5
timeout 300 python tools/closedloop_bench.py --periods 200 > gpurun_out/cl_single.json 2> gpurun_out/cl_single.err; cat gpurun_out/cl_single.json; tail -3 gpurun_out/cl_single.err
timeout 300 python tools/closedloop_bench.py --dof 12 --N 512 --K 32 --T 50 --p 3 --fleet 64 --periods 20 > gpurun_out/cl_fleet.json 2> gpurun_out/cl_fleet.err; cat gpurun_out/cl_fleet.json; tail -3 gpurun_out/cl_fleet.err
