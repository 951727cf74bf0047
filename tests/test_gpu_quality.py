"""Statistical quality gate of the production RNG path (SPEC.md:665,
acceptance #9): on a fixed-x0 linear pendulum problem
(T = 50, p = 3), EMPC with 1024 sims, 64 parents and 200 generations must come
within 5 % of the small-parameterized convex QP optimum in >= 95 % of 20
seeds.  The in-kernel counter-based Philox streams replace numpy's Philox
(K/empc.py:68-70), so this is the acceptance test of that replacement, run
through the benched device path (per-generation launches for n = 2).

The problem: the reference's g = 0 pendulum (K/dynamics.py:33-75 defaults,
gravity 0) linearized at rest and discretized exactly at dt = 0.01, the
closed-loop template weights Q = diag(10, 0.1), R = 0.01, |u| <= 25
(K/bench.py:360-376), goal angle 0.5 rad from rest.  The QP optimum is the
oracle's exact box-QP minimum of the condensed quadratic (K/condense.py:268-274).
"""

import numpy as np
import pytest

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import dynamics as D
from oracle import empc_oracle as O

pytestmark = pytest.mark.gpu


def _linear_pendulum():
    plant = D.Pendulum(D.PendulumParams(gravity=0.0))
    model = D.discretize(D.linearize(plant.ode, np.zeros(2), np.zeros(1)), 0.01)
    return P.MpcSpec(model, 50, Q=np.diag([10.0, 0.1]), R=0.01 * np.eye(1), x_goal=np.array([0.5, 0.0]),
                     u_goal=np.zeros(1), u_min=np.array([-25.0]), u_max=np.array([25.0]))


def test_convergence_to_qp_optimum_over_20_seeds():
    spec = _linear_pendulum()
    sched = P.KnotSchedule(50, 3)
    x0 = np.zeros(2)
    opt = O.qp_optimum(O.Problem.from_spec(spec), 3, x0)
    ratios = []
    for seed in range(20):
        st = P.EmpcSettings(num_sims=1024, num_parents=64, generations=200, seed=seed)
        res = P.solve_empc(spec, sched, st, x0)
        ratios.append(res.best_cost / opt)
    ratios = np.array(ratios)
    assert np.all(ratios >= 1.0 - 1e-5), ratios.min()  # never below the convex optimum
    assert np.mean(ratios <= 1.05) >= 0.95, np.sort(ratios)
