"""Host-side profile of the public-API solve (bench e2e path), cold C3 solves:
wall time per call vs the device time, and where the host time goes."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2001_04931_b200 as P  # noqa: E402
from paper_2001_04931_b200 import workloads as W  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
w = W.WORKLOADS[cfg]
specs, x0s = W.build(w)
st = w.settings()
sched = w.schedule()
for _ in range(5):
    P.solve_empc(specs[0], sched, st, x0s[0])
t = []
for _ in range(200):
    t0 = time.perf_counter()
    r = P.solve_empc(specs[0], sched, st, x0s[0])
    t.append(time.perf_counter() - t0)
t.sort()
print(f"{cfg} e2e median {t[len(t)//2]*1e3:.4f} ms  min {t[0]*1e3:.4f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    P.solve_empc(specs[0], sched, st, x0s[0])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)

# breakdown: public API vs bare empc_run vs device time
import ctypes as C  # noqa: E402

from paper_2001_04931_b200 import _native as nat  # noqa: E402
from paper_2001_04931_b200 import empc as E  # noqa: E402

ctx = E._spec_context(specs[0], sched, st)
sigma = E._mutation_sigma(specs[0], st, x0s[0])
a = nat.empc_run_args()
x0c, sg = nat.f64(x0s[0][None]), nat.f64(sigma[None])
u = np.empty((1, w.m)) if False else None
import numpy as np  # noqa: E402

u, best, bc, bi = np.empty((1, w.m)), np.empty((1, w.p, w.m)), np.empty(1), np.empty(1, np.int32)
slot = ctx.slot()
a.init, a.rescore, a.evolves, a.slot_in, a.slot_out = 1, 0, w.G - 1, -1, slot.id
a.generation0, a.seed, a.mutation_prob, a.crossover_prob = 1, st.seed, st.mutation_prob, st.crossover_prob
a.x0, a.sigma = nat.dptr(x0c), nat.dptr(sg)
a.u_out, a.best_out, a.best_cost, a.best_index = nat.dptr(u), nat.dptr(best), nat.dptr(bc), nat.iptr(bi)
for variant in ("slot", "noslot"):
    a.slot_out = slot.id if variant == "slot" else -1
    tt = []
    for _ in range(300):
        t0 = time.perf_counter()
        ctx.h.call("empc_run", C.byref(a))
        tt.append(time.perf_counter() - t0)
    tt.sort()
    print(f"bare empc_run ({variant}) median {tt[len(tt)//2]*1e3:.4f} ms")
ms = (C.c_float * 100)()
ctx.h.call("empc_time_device", C.byref(a), 100, 0, ms, None, None, None)
v = sorted(ms)
print(f"device (graph, no flush) median {v[50]:.4f} ms")
ctx.h.call("empc_time_device", C.byref(a), 100, 1, ms, None, None, None)
v = sorted(ms)
print(f"device (graph, L2 flushed) median {v[50]:.4f} ms")
tt = []
for _ in range(300):
    t0 = time.perf_counter()
    E._spec_context(specs[0], sched, st)
    tt.append(time.perf_counter() - t0)
tt.sort()
print(f"_spec_context median {tt[150]*1e6:.1f} us")
