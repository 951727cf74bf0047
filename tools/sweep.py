"""Run bench.py once per environment setting and print ms_per_step and the
path taken.  Usage: python tools/sweep.py CONFIG 'ENV=..,ENV2=..' ['...']"""
import json
import os
import subprocess
import sys

cfg = sys.argv[1]
for spec in sys.argv[2:] or [""]:
    env = dict(os.environ)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "50", "--warmup", "5",
                        "--no-cpu-baseline"], env=env, capture_output=True, text=True, timeout=300)
    try:
        d = json.loads(r.stdout.strip().splitlines()[-1])
        print(f"{cfg} [{spec}] {d['ms_per_step'] * 1e3:.1f} us | {d['config']['kernel_variant'][-80:]}", flush=True)
    except Exception:
        print(f"{cfg} [{spec}] FAILED rc={r.returncode}: {r.stderr[-300:]}", flush=True)
