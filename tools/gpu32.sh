for c in c1 c2; do timeout 300 python bench.py --config $c --steps 100 --warmup 10 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
for c in c1 c2 c3; do timeout 300 python bench.py --config $c --scorer condensed --steps 50 --warmup 5 > gpurun_out/cond_$c.json 2> gpurun_out/cond_$c.err; done
timeout 600 python bench.py --config c4 --scorer condensed --steps 10 --warmup 3 --cpu-sample-s 20 > gpurun_out/cond_c4.json 2> gpurun_out/cond_c4.err
timeout 900 python bench.py --config c5 --scorer condensed --steps 5 --warmup 3 --cpu-sample-s 10 > gpurun_out/cond_c5.json 2> gpurun_out/cond_c5.err
timeout 300 python tools/closedloop_bench.py --dof 12 --N 512 --K 32 --T 50 --p 3 --fleet 1024 --periods 20 > gpurun_out/cl_fleet.json 2>&1
