"""Randomised shapes through every execution path (resident small solve,
persistent solve, per-generation launches): the final population's costs
equal the FP64 oracle's rollout of its candidates (1e-5), the elite block
is sorted ascending and holds the best candidate, every knot is inside the
input box, and u / best / best_cost are consistent (K/empc.py:211-236)."""

import numpy as np
import pytest

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import _native as nat
from paper_2001_04931_b200 import empc as E
from oracle import empc_oracle as O

pytestmark = pytest.mark.gpu

PATHS = {
    "default": {},
    "small": {nat.EMPC_OPT_SMALL_SOLVE: 1},
    "persistent": {nat.EMPC_OPT_SMALL_SOLVE: 0, nat.EMPC_OPT_PERSISTENT: 1},
    "launches": {nat.EMPC_OPT_SMALL_SOLVE: 0, nat.EMPC_OPT_PERSISTENT: 0},
}
RESET = {nat.EMPC_OPT_SMALL_SOLVE: -1, nat.EMPC_OPT_PERSISTENT: -1}


def _random_problem(rng, n, m, T, dense_r):
    A = np.eye(n) + 0.02 * rng.standard_normal((n, n))
    B = 0.05 * rng.standard_normal((n, m))
    w = 0.01 * rng.standard_normal(n)
    if dense_r:
        Mr = rng.standard_normal((m, m))
        R = Mr @ Mr.T / m + 0.1 * np.eye(m)
    else:
        R = np.diag(rng.uniform(0.01, 0.1, m))
    spec = P.MpcSpec(P.DiscreteLinearModel(A, B, w, 0.01), T, Q=np.diag(rng.uniform(0.1, 10.0, n)), R=R,
                     x_goal=rng.uniform(-1, 1, n), u_goal=0.1 * rng.standard_normal(m), u_min=-np.ones(m),
                     u_max=np.ones(m))
    return spec, rng.uniform(-1, 1, n)


SHAPES = [  # n, m, T, p, N, K, G, dense R
    (2, 1, 20, 3, 64, 8, 4, False),
    (4, 2, 20, 2, 100, 6, 5, False),
    (3, 2, 15, 1, 50, 5, 3, True),
    (8, 3, 25, 8, 128, 16, 3, False),
    (12, 6, 30, 3, 512, 32, 3, True),
    (24, 12, 20, 4, 700, 40, 3, False),
    (48, 24, 12, 4, 2048, 128, 3, False),
    (7, 4, 40, 6, 300, 300, 2, False),  # K == N
]


@pytest.mark.parametrize("shape", SHAPES, ids=[f"n{s[0]}_m{s[1]}_T{s[2]}_p{s[3]}_N{s[4]}" for s in SHAPES])
@pytest.mark.parametrize("path", sorted(PATHS))
def test_random_shapes_every_path(shape, path):
    n, m, T, p, N, K, G, dense_r = shape
    rng = np.random.default_rng(hash(shape) % (2 ** 32))
    spec, x0 = _random_problem(rng, n, m, T, dense_r)
    sched = P.KnotSchedule(T, p)
    st = P.EmpcSettings(num_sims=N, num_parents=K, generations=G, seed=3)
    ctx = E._spec_context(spec, sched, st)
    try:
        for opt, val in PATHS[path].items():
            ctx.h.set_option(opt, val)
        res = P.solve_empc(spec, sched, st, x0)
        desc = ctx.h.describe()
    finally:
        for opt, val in RESET.items():
            ctx.h.set_option(opt, val)
    cands, costs = res.population.candidates, res.population.costs
    pr = O.Problem.from_spec(spec)
    np.testing.assert_allclose(costs, O.rollout_costs(cands, pr, x0), rtol=1e-5, err_msg=desc)
    Kc = min(K, N)
    assert np.all(np.diff(costs[:Kc]) >= 0), desc
    assert res.best_cost == np.min(costs)
    np.testing.assert_array_equal(res.best, cands[int(np.argmin(costs))])
    np.testing.assert_array_equal(res.u, res.best[0])
    assert np.all(cands >= -1.0) and np.all(cands <= 1.0)
    if path == "small" and n <= 8 and N <= 4096:
        assert "resident single-CTA" in desc, desc
    if path == "launches":
        assert "per-generation" in desc, desc


WARM_SHAPES = [SHAPES[1], SHAPES[4], SHAPES[6]]


@pytest.mark.parametrize("shape", WARM_SHAPES, ids=[f"n{s[0]}_N{s[4]}" for s in WARM_SHAPES])
@pytest.mark.parametrize("path", sorted(PATHS))
def test_warm_start_reads_the_input_population_in_place(shape, path):
    """Warm public-API solves read `prev` straight from its slot inside the
    graph (no copy before it): `prev` stays untouched, the result is the
    oracle-consistent re-score + G generations, and repeating the call with
    the same `prev` gives the same bits (both slot alternations)."""
    n, m, T, p, N, K, G, dense_r = shape
    rng = np.random.default_rng(17 + n)
    spec, x0 = _random_problem(rng, n, m, T, dense_r)
    sched = P.KnotSchedule(T, p)
    st = P.EmpcSettings(num_sims=N, num_parents=K, generations=G, seed=4)
    ctx = E._spec_context(spec, sched, st)
    pr = O.Problem.from_spec(spec)
    try:
        for opt, val in PATHS[path].items():
            ctx.h.set_option(opt, val)
        cold = P.solve_empc(spec, sched, st, x0)
        prev = cold.population
        before = (prev.candidates.copy(), prev.costs.copy())
        x1 = x0 + 0.05
        runs = [P.solve_empc(spec, sched, st, x1, prev) for _ in range(3)]
        desc = ctx.h.describe()
    finally:
        for opt, val in RESET.items():
            ctx.h.set_option(opt, val)
    np.testing.assert_array_equal(prev.candidates, before[0])
    np.testing.assert_array_equal(prev.costs, before[1])
    for r in runs[1:]:
        np.testing.assert_array_equal(r.population.candidates, runs[0].population.candidates)
        np.testing.assert_array_equal(r.population.costs, runs[0].population.costs)
        assert r.best_cost == runs[0].best_cost
    c, k = runs[0].population.candidates, runs[0].population.costs
    np.testing.assert_allclose(k, O.rollout_costs(c, pr, x1), rtol=1e-5, err_msg=desc)
    assert np.all(np.diff(k[:K]) >= 0), desc
    assert runs[0].best_cost == np.min(k)
    assert runs[0].population.generation == prev.generation + G
