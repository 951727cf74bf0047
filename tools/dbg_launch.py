import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import _native as nat, empc as E, workloads as W
w = W.WORKLOADS["c3"]
specs, x0s = W.build(w)
st = w.settings()
def attempt(tag, occ=None, score=False, variant=None, rollout=False):
    E._contexts.clear()
    ctx = E._spec_context(specs[0], w.schedule(), st)
    if variant is not None: ctx.h.set_variant(variant)
    if occ is not None: ctx.h.set_occupancy(occ)
    sigma = E._mutation_sigma(specs[0], st, x0s[0])[None]
    a = nat.empc_run_args()
    x0c, sg = nat.f64(x0s), nat.f64(sigma)
    a.init, a.rescore, a.evolves, a.slot_in, a.slot_out = 1, 0, w.G - 1, -1, -1
    a.generation0, a.seed, a.mutation_prob, a.crossover_prob = 1, st.seed, st.mutation_prob, st.crossover_prob
    a.x0, a.sigma = nat.dptr(x0c), nat.dptr(sg)
    ms = (C.c_float * 3)()
    rms, nr, nl = C.c_float(), C.c_int32(), C.c_int32()
    try:
        ctx.h.call("empc_time_device", C.byref(a), 3, 1, ms, C.byref(rms) if rollout else None, C.byref(nr), C.byref(nl))
        print(tag, "ok", list(ms), rms.value)
    except Exception as e:
        print(tag, "ERR", e)
attempt("plain")
attempt("plain-rollout", rollout=True)
attempt("occ1", occ=1)
attempt("v0", variant=0)
attempt("v7", variant=7)
r = P.solve_empc(specs[0], w.schedule(), st, x0s[0]); print("solve ok", r.best_cost)
