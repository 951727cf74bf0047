# C3 persistent-solve phase timers with the half-K matvec.
EMPC_PHASES=1 timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c3ph.json 2> gpurun_out/c3ph.err; grep -v "^$" gpurun_out/c3ph.err | tail -6
