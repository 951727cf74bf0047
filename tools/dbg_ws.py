"""Debug helper: C3 populations after G generations through the per-launch
path and the persistent path (variant / predraw from the environment)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import empc as E, workloads as W, _native as nat
w = W.WORKLOADS["c3"]
specs, x0s = W.build(w)
G = int(sys.argv[1]) if len(sys.argv) > 1 else 3
st = w.settings(generations=G)
ctx = E._spec_context(specs[0], w.schedule(), st)
out = {}
for mode in (0, 1):
    ctx.h.set_option(nat.EMPC_OPT_PERSISTENT, mode)
    ctx.h.set_option(nat.EMPC_OPT_HALF_K, 0)
    r = P.solve_empc(specs[0], w.schedule(), st, x0s[0])
    out[mode] = (r.population.candidates.copy(), r.population.costs.copy(), ctx.h.describe())
    print(mode, out[mode][2][-90:])
a, b = out[0], out[1]
rows = np.flatnonzero(np.any(a[0] != b[0], axis=(1, 2)))
print("G", G, "mismatched rows", rows.size, rows[:20], "costs equal", np.array_equal(a[1], b[1]))
