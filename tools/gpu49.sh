# Final check of the shipped tree: GPU tests, smoke, default bench line; C5 phase breakdown.
timeout 900 python -m pytest tests/ -q -m gpu --timeout 300 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/final_c3.json 2> gpurun_out/final_c3.err; head -c 300 gpurun_out/final_c3.json; echo
EMPC_PHASES=1 timeout 600 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5ph.json 2> gpurun_out/c5ph.err; grep -i "phase\|step\|prologue" gpurun_out/c5ph.err | tail -8
