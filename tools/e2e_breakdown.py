"""Where the time of one public-API solve_empc call goes (host side), C3."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import empc as E, workloads as W
w = W.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
specs, x0s = W.build(w)
spec, sched, st, x0 = specs[0], w.schedule(), w.settings(), x0s[0]
for _ in range(20):
    P.solve_empc(spec, sched, st, x0)
t = {"spec_context": [], "sigma": [], "run": [], "total": []}
for _ in range(200):
    a = time.perf_counter()
    ctx = E._spec_context(spec, sched, st)
    b = time.perf_counter()
    sg = E._mutation_sigma(spec, st, x0)
    c = time.perf_counter()
    E._run(ctx, st, x0, sg, init=True, rescore=False, evolves=st.generations - 1, gen0=1)
    d = time.perf_counter()
    t["spec_context"].append(b - a); t["sigma"].append(c - b); t["run"].append(d - c); t["total"].append(d - a)
print({k: round(float(np.median(v)) * 1e6, 1) for k, v in t.items()}, "us (median)")
