"""Timing of the batched device plant model against the host
restatement of linearize + discretize / RK4 (K/dynamics.py:241-330).

    python tools/plant_bench.py      -> one JSON line per case
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2001_04931_b200 import dynamics as D  # noqa: E402


def case(links, count, host_sample=8):
    plant = D.NLinkArm(D.NLinkParams(links=links))
    rng = np.random.default_rng(0)
    xs = np.concatenate([rng.uniform(-np.pi, np.pi, (count, links)), np.zeros((count, links))], axis=1)
    us = np.zeros((count, links))
    D.linearize_discretize(plant, xs[:2], us[:2], 0.01)  # warm-up (context, module load)
    D.integrate_batch(plant, xs[:2], us[:2], 0.01, 10)
    reps = 5
    t0 = time.perf_counter()
    for _ in range(reps):
        D.linearize_discretize(plant, xs, us, 0.01)
    dev_ld = (time.perf_counter() - t0) / reps
    t0 = time.perf_counter()
    for _ in range(reps):
        D.integrate_batch(plant, xs, us, 0.01, 10)
    dev_rk = (time.perf_counter() - t0) / reps
    k = min(host_sample, count)
    t0 = time.perf_counter()
    for i in range(k):
        D.discretize(D.linearize(plant.ode, xs[i], us[i]), 0.01)
    host_ld = (time.perf_counter() - t0) / k
    t0 = time.perf_counter()
    for i in range(k):
        D.integrate(plant.ode, xs[i], us[i], 0.01, 10)
    host_rk = (time.perf_counter() - t0) / k
    print(json.dumps({"what": "plant linearize+discretize(exact) / RK4 period", "links": links, "instances": count,
                      "device_linearize_discretize_ms": dev_ld * 1e3, "device_rk4_ms": dev_rk * 1e3,
                      "host_linearize_discretize_ms_per_instance": host_ld * 1e3,
                      "host_rk4_ms_per_instance": host_rk * 1e3,
                      "host_estimate_all_instances_ms": (host_ld + host_rk) * count * 1e3,
                      "note": "device times include H2D of x,u and D2H of Ad,Bd,wd / x (host arrays in and out)"}))


if __name__ == "__main__":
    case(2, 1)
    case(24, 1)
    case(48, 1)
    case(12, 8192)
    case(24, 1024)
