"""Small driver for ncu: a few cold solves of one workload through the public API."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variant = int(sys.argv[3]) if len(sys.argv) > 3 else -1
w = W.WORKLOADS[cfg]
if w.instances > 1:
    w = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, instances=int(os.environ.get("PROF_INSTANCES", 512)))
specs, x0s = W.build(w)
st = w.settings()
if w.instances > 1:
    b = P.EmpcBatch(specs, w.schedule(), st)
    if variant >= 0:
        b.ctx.h.set_variant(variant)
    for _ in range(reps):
        r = b.solve(x0s)
    print(cfg, "best_cost[0]", r.best_cost[0], b.ctx.h.describe())
else:
    from paper_2001_04931_b200 import empc as E
    ctx = E._spec_context(specs[0], w.schedule(), st)
    if variant >= 0:
        ctx.h.set_variant(variant)
    for _ in range(reps):
        r = P.solve_empc(specs[0], w.schedule(), st, x0s[0])
    print(cfg, "best_cost", r.best_cost, ctx.h.describe())
