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
