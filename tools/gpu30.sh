timeout 600 python -m pytest tests/test_gpu_plant.py tests/test_closedloop.py -x -q -m gpu --timeout 200 2>&1 | tail -15
timeout 300 python tools/closedloop_bench.py --dof 12 --N 512 --K 32 --T 50 --p 3 --fleet 64 --periods 20 2>&1 | tail -2
