"""Closed-loop EMPC timing: steady-state warm solve latency at
100 Hz with the population resident on the GPU, next to the host time the
loop spends relinearizing/discretizing and integrating the plant.

    python tools/closedloop_bench.py [--dof 24] [--periods 200] [--fleet 0]

Prints one JSON line.  Arm: the C3 settings (N=4096, K=256, G=10, T=50, p=4)
on a 24-DoF N-link arm stepping to a random joint goal (K/bench.py:396-412).
``--fleet I`` runs I such plants through ClosedLoopFleet instead.
"""

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import paper_2001_04931_b200 as P  # noqa: E402
from paper_2001_04931_b200 import closedloop as CL  # noqa: E402
from paper_2001_04931_b200 import dynamics as D  # noqa: E402


def template(plant, T, umax):
    nj = plant.m
    clin = D.linearize(plant.ode, np.zeros(plant.n), np.zeros(nj))
    return P.MpcSpec(D.discretize(clin, 0.01), T, Q=np.diag([10.0] * nj + [0.1] * nj), R=0.01 * np.eye(nj),
                     x_goal=np.zeros(plant.n), u_goal=np.zeros(nj), u_min=-umax * np.ones(nj),
                     u_max=umax * np.ones(nj))


def q(a):
    return [float(v) * 1e3 for v in np.percentile(a, [25, 50, 75])]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dof", type=int, default=24)
    ap.add_argument("--periods", type=int, default=200)
    ap.add_argument("--N", type=int, default=4096)
    ap.add_argument("--K", type=int, default=256)
    ap.add_argument("--G", type=int, default=10)
    ap.add_argument("--T", type=int, default=50)
    ap.add_argument("--p", type=int, default=4)
    ap.add_argument("--fleet", type=int, default=0)
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    st = P.EmpcSettings(num_sims=a.N, num_parents=a.K, generations=a.G, seed=1)
    ctl = CL.Controller("empc", p=a.p, empc=st)
    plant = D.NLinkArm(D.NLinkParams(links=a.dof))
    tpl = template(plant, a.T, 2.0)
    n = plant.n
    if a.fleet:
        goals = np.concatenate([rng.uniform(-0.5, 0.5, (a.fleet, a.dof)), np.zeros((a.fleet, a.dof))], axis=1)
        fleet = CL.ClosedLoopFleet([plant] * a.fleet, ctl, tpl, goals, rate=100.0)
        x = np.zeros((a.fleet, n))
        solve, host = [], []
        for i in range(a.periods):
            t0 = time.perf_counter()
            x, u, ts = fleet.step(x)
            host.append(time.perf_counter() - t0 - ts)
            solve.append(ts)
        err = float(np.abs(x[:, :a.dof] - goals[:, :a.dof]).max())
        print(json.dumps({"what": "closed-loop fleet", "instances": a.fleet, "dof": a.dof, "periods": a.periods,
                          "N": a.N, "K": a.K, "G": a.G, "T": a.T, "p": a.p,
                          "warm_solve_ms_q1_med_q3": q(solve[1:]), "cold_solve_ms": solve[0] * 1e3,
                          "host_linearize_discretize_integrate_ms_median": float(np.median(host)) * 1e3,
                          "final_max_joint_error": err}))
        return
    goal = np.concatenate([rng.uniform(-0.5, 0.5, a.dof), np.zeros(a.dof)])
    x = np.zeros(n)
    pop = None
    solve, lin, integ = [], [], []
    sched = P.KnotSchedule(a.T, a.p)
    from dataclasses import replace
    for i in range(a.periods):
        t0 = time.perf_counter()
        spec = replace(tpl, model=D.discretize(D.linearize(plant.ode, x, np.zeros(a.dof)), 0.01), x_goal=goal)
        t1 = time.perf_counter()
        r = P.solve_empc(spec, sched, st, x, prev=pop)
        t2 = time.perf_counter()
        pop = r.population
        x = D.integrate(plant.ode, x, np.clip(r.u, spec.u_min, spec.u_max), 0.01)
        t3 = time.perf_counter()
        lin.append(t1 - t0)
        solve.append(t2 - t1)
        integ.append(t3 - t2)
    print(json.dumps({"what": "closed-loop single plant", "dof": a.dof, "periods": a.periods, "rate_hz": 100,
                      "N": a.N, "K": a.K, "G": a.G, "T": a.T, "p": a.p,
                      "warm_solve_ms_q1_med_q3": q(solve[1:]), "cold_solve_ms": solve[0] * 1e3,
                      "host_linearize_discretize_ms_median": float(np.median(lin)) * 1e3,
                      "host_rk4_ms_median": float(np.median(integ)) * 1e3,
                      "final_max_joint_error": float(np.abs(x[:a.dof] - goal[:a.dof]).max()),
                      "solve_api": "solve_empc(prev=population) -- population resident on the GPU"}))


if __name__ == "__main__":
    main()
