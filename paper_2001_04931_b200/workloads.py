"""Benchmark workloads C1-C5 (BASELINE.json configs, SURVEY.md §8 glossary).

Synthetic systems follow the reference harness recipe (SURVEY.md §8d,
K/bench.py:360-412, K/bench.py:571-606): ``NLinkArm(D)`` with default
parameters (1 kg, 0.25 m, b = 0.01, g = 0), start and goal joint angles
uniform in [-pi, pi] at rest, linearized at the start with zero torque and
discretized exactly at dt = 0.01; Q = diag(10 I_D, 0.1 I_D), R = 0.01 I_D,
torque bounds +-2.  System seed 0 for C1-C4, instance seed i for C5;
EmpcSettings.seed = 1.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dynamics import NLinkArm, NLinkParams, discretize, linearize
from .empc import EmpcSettings
from .param import KnotSchedule
from .spec import MpcSpec


@dataclass(frozen=True)
class Workload:
    name: str
    dof: int
    T: int
    p: int
    N: int
    K: int
    G: int
    instances: int = 1

    @property
    def n(self):
        return 2 * self.dof

    @property
    def m(self):
        return self.dof

    @property
    def scored_per_solve(self) -> int:
        """Candidates scored by one cold solve, all instances."""
        return (self.N + (self.G - 1) * (self.N - self.K)) * self.instances

    @property
    def cand_steps_per_solve(self) -> int:
        return self.scored_per_solve * self.T

    @property
    def flop_per_candidate(self) -> int:
        """Algorithmic FP32 work per scored candidate, 2 T n^2 + 2 p n m."""
        return 2 * self.T * self.n ** 2 + 2 * self.p * self.n * self.m

    def settings(self, **kw) -> EmpcSettings:
        base = dict(num_sims=self.N, num_parents=self.K, generations=self.G, seed=1)
        base.update(kw)
        return EmpcSettings(**base)

    def schedule(self) -> KnotSchedule:
        return KnotSchedule(self.T, self.p)


WORKLOADS = {
    "c1": Workload("c1", 2, 20, 2, 100, 6, 10),
    "c2": Workload("c2", 6, 50, 3, 1024, 64, 10),
    "c3": Workload("c3", 24, 50, 4, 4096, 256, 10),
    "c4": Workload("c4", 48, 200, 5, 16384, 1024, 10),
    "c5": Workload("c5", 12, 50, 3, 512, 32, 10, instances=8192),
}


def nlink_problem(dof: int, T: int, seed: int, dt: float = 0.01):
    """(spec, x0) for one synthetic N-link system (reference recipe)."""
    plant = NLinkArm(NLinkParams(links=dof))
    rng = np.random.default_rng(seed)
    q0 = rng.uniform(-np.pi, np.pi, dof)
    qg = rng.uniform(-np.pi, np.pi, dof)
    x0 = np.concatenate([q0, np.zeros(dof)])
    xg = np.concatenate([qg, np.zeros(dof)])
    model = discretize(linearize(plant.ode, x0, np.zeros(dof)), dt)
    spec = MpcSpec(model, T, Q=np.diag([10.0] * dof + [0.1] * dof), R=0.01 * np.eye(dof), x_goal=xg,
                   u_goal=np.zeros(dof), u_min=np.full(dof, -2.0), u_max=np.full(dof, 2.0))
    return spec, x0


def build(w: Workload, first_instance: int = 0, count: int | None = None):
    """Specs and start states of a workload; instances [first, first+count)."""
    if w.instances == 1:
        spec, x0 = nlink_problem(w.dof, w.T, 0)
        return [spec], x0[None]
    count = w.instances - first_instance if count is None else count
    specs, x0s = [], []
    for i in range(first_instance, first_instance + count):
        s, x = nlink_problem(w.dof, w.T, i)
        specs.append(s)
        x0s.append(x)
    return specs, np.stack(x0s)
