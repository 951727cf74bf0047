for x in 0 1 2; do
  EMPC_TC_EXP=$x EMPC_PHASES=1 timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --tensor-cores on > gpurun_out/tcx_$x.json 2> gpurun_out/tcx_$x.err
  echo "exp $x"; grep -E "tc step" gpurun_out/tcx_$x.err | tail -1
  python -c "import json;d=json.load(open('gpurun_out/tcx_$x.json'));print(d['roofline']['rollout_ms_per_launch'])"
done
