"""Fixed (prologue) vs per-step cost of the rollout kernel: score N candidates
of a C3-shaped system at several horizons.  Usage: python tools/steps.py [variant]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2001_04931_b200 import _native as nat
from paper_2001_04931_b200 import empc as E
from paper_2001_04931_b200 import workloads as W

dof = int(os.environ.get("DOF", 24))
N = int(os.environ.get("NSC", 3840))
variant = int(sys.argv[1]) if len(sys.argv) > 1 else -1
for T in (4, 26, 50, 98):
    spec, x0 = W.nlink_problem(dof, T, 0)
    p = 4
    ctx = E._context(2 * dof, dof, T, p, 1, 1, 1, False, "fp32")
    if variant >= 0:
        ctx.h.set_variant(variant)
    ctx.set_problems(E._problem_arrays(spec))
    cands = np.random.default_rng(0).uniform(-2, 2, size=(N, p, dof))
    costs = np.empty(N)
    args = (nat.dptr(nat.f64(x0)), N, nat.dptr(nat.f64(cands)), nat.dptr(costs))
    for _ in range(3):
        ctx.h.call("empc_score", *args)
    # time with the host clock around synchronous calls minus the transfer-only call (num=0 not possible):
    # use many reps and CUDA's own sync; transfers are small (N*p*m doubles)
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        ctx.h.call("empc_score", *args)
    dt = (time.perf_counter() - t0) / reps
    print(f"T={T:4d} score {N} cands: {dt*1e6:8.1f} us/call  ({ctx.h.describe()[:80]})", flush=True)
