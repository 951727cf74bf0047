"""Variant sweep: for each compiled rollout variant, check scoring parity
against the oracle and time the device-resident cold solve and the mean
rollout launch.  Usage: python tools/tune.py c3 [reps]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import _native as nat
from paper_2001_04931_b200 import empc as E
from paper_2001_04931_b200 import workloads as W
from oracle import empc_oracle as O

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
w = W.WORKLOADS[cfg]
if w.instances > 1:
    w = W.Workload(w.name, w.dof, w.T, w.p, w.N, w.K, w.G, instances=int(os.environ.get("TUNE_INSTANCES", 1024)))
specs, x0s = W.build(w)
st = w.settings()
if w.instances > 1:
    b = P.EmpcBatch(specs, w.schedule(), st)
    ctx, sigma = b.ctx, b.sigma(x0s)
else:
    ctx = E._spec_context(specs[0], w.schedule(), st)
    sigma = E._mutation_sigma(specs[0], st, x0s[0])[None]
a = nat.empc_run_args()
x0c, sg = nat.f64(x0s), nat.f64(sigma)
a.init, a.rescore, a.evolves, a.slot_in, a.slot_out = 1, 0, w.G - 1, -1, -1
a.generation0, a.seed, a.mutation_prob, a.crossover_prob = 1, st.seed, st.mutation_prob, st.crossover_prob
a.x0, a.sigma = nat.dptr(x0c), nat.dptr(sg)
pr = O.Problem.from_spec(specs[0])
rng = np.random.default_rng(0)
cands = rng.uniform(pr.u_min, pr.u_max, size=(64, w.p, w.m))
want = O.rollout_costs(cands, pr, x0s[0])
sctx = E._context(w.n, w.m, w.T, w.p, 1, 1, 1, False, "fp32")
sctx.set_problems(E._problem_arrays(specs[0]))
rows = []
cps_list = [int(x) for x in os.environ.get("TUNE_CPS", "0").split(",")]
only = os.environ.get("TUNE_VARIANTS")
vlist = [int(x) for x in only.split(",")] if only else range(ctx.h.num_variants())
for v, cps in [(v, c) for v in vlist for c in cps_list]:
    try:
        ctx.h.set_variant(v)
        sctx.h.set_variant(v)
        ctx.h.set_occupancy(cps)
    except ValueError:
        continue
    try:
        costs = np.empty(64)
        sctx.h.call("empc_score", nat.dptr(nat.f64(x0s[0])), 64, nat.dptr(nat.f64(cands)), nat.dptr(costs))
        err = float(np.max(np.abs(costs - want) / np.abs(want)))
        ms = (C.c_float * reps)()
        rms, nr, nl = C.c_float(), C.c_int32(), C.c_int32()
        ctx.h.call("empc_time_device", C.byref(a), 3, 1, ms, None, C.byref(nr), C.byref(nl))
        ctx.h.call("empc_time_device", C.byref(a), reps, 1, ms, C.byref(rms), C.byref(nr), C.byref(nl))
        t = sorted(list(ms))
        flop = w.flop_per_candidate * w.scored_per_solve / nr.value
        row = dict(variant=v, cps=cps, desc=ctx.h.describe(), solve_ms=t[len(t) // 2], rollout_ms=rms.value,
                   tflops=flop / (rms.value * 1e-3) / 1e12, rel_err=err)
    except Exception as e:  # noqa: BLE001
        row = dict(variant=v, cps=cps, error=str(e)[:200])
    rows.append(row)
    print(json.dumps(row), flush=True)
ctx.h.set_variant(-1)
