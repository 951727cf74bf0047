"""Condensed scorer: the reference's own knot-space quadratic
(K/empc.py:122-152, built by K/condense.py:268-274) evaluated on the GPU.

Tolerances: FP64 device mode 1e-11 relative against the reference's FP64
condensed costs (same function, different summation order); FP32 populations
1e-5 (the candidates are rounded to FP32 before scoring, the quadratic form
itself runs in FP64).
"""

import numpy as np
import pytest

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import shard as SH
from oracle import empc_oracle as O
from tests import golden as G

pytestmark = pytest.mark.gpu

RTOL64 = 1e-11
RTOL32 = 1e-5


def _sched(g):
    return P.KnotSchedule(int(g["T"]), int(g["p"]))


@pytest.mark.parametrize("name", ["spec2", "c1", "c2", "c3s", "dense"])
@pytest.mark.parametrize("precision,rtol", [("fp64", RTOL64), ("fp32", RTOL32)])
def test_condensed_scorer_matches_reference(name, precision, rtol):
    g = G.load("score_" + name)
    got = P.CostModel(G.spec(g), _sched(g), g["x0"], precision=precision, scorer="condensed")(g["cands"])
    np.testing.assert_allclose(got, g["cost_condensed"], rtol=rtol)


@pytest.mark.parametrize("num", [1, 3, 33, 200, 1000])
def test_condensed_ragged_batches(num):
    g = G.load("score_c2")
    pr = G.problem(g)
    rng = np.random.default_rng(num)
    cands = rng.uniform(pr.u_min, pr.u_max, size=(num, int(g["p"]), pr.m))
    got = P.CostModel(G.spec(g), _sched(g), g["x0"], precision="fp64", scorer="condensed")(cands)
    np.testing.assert_allclose(got, O.CostModel(pr, int(g["p"]), g["x0"])(cands), rtol=RTOL64)


@pytest.mark.parametrize("n,m,p,T,dense", [(6, 40, 5, 12, False), (5, 3, 64, 70, True), (64, 8, 3, 30, False)])
def test_condensed_shapes(n, m, p, T, dense):
    """Long knot vectors (P streamed from L2 when it does not fit in shared
    memory), dense Q, large state: against the oracle's condensed model."""
    rng = np.random.default_rng(n * 1000 + m)
    A = rng.normal(size=(n, n)) * (0.9 / np.sqrt(n)) + 0.5 * np.eye(n)
    B = rng.normal(size=(n, m)) * 0.1
    if dense:
        L = rng.normal(size=(n, n))
        Q = L @ L.T / n + np.eye(n)
    else:
        Q = np.diag(rng.uniform(0.1, 10.0, n))
    R = np.diag(rng.uniform(0.01, 0.1, m))
    spec = P.MpcSpec(P.DiscreteLinearModel(A, B, rng.normal(size=n) * 0.01, 0.01), T, Q, R,
                     rng.normal(size=n), np.zeros(m), -np.ones(m), np.ones(m))
    x0 = rng.normal(size=n)
    cands = rng.uniform(-1, 1, size=(300, p, m))
    got = P.CostModel(spec, P.KnotSchedule(T, p), x0, precision="fp64", scorer="condensed")(cands)
    pr = O.Problem.from_spec(spec)
    want = O.CostModel(pr, p, x0)(cands)
    np.testing.assert_allclose(got, want, rtol=1e-10)
    roll = O.rollout_costs(cands, pr, x0)
    np.testing.assert_allclose(got, roll, rtol=1e-9)


def test_state_bounded_spec_rolls_out():
    """K/empc.py:138: specs with state bounds keep the rollout."""
    g = G.load("bounded")
    s2 = G.load("score_spec2")
    spec = G.spec(s2)
    bounded = P.MpcSpec(spec.model, 20, spec.Q, spec.R, spec.x_goal, spec.u_goal, spec.u_min, spec.u_max,
                        x_min=-10.0 * np.ones(2), x_max=10.0 * np.ones(2))
    got = P.CostModel(bounded, P.KnotSchedule(20, int(s2["p"])), s2["x0"], precision="fp64",
                      scorer="condensed")(g["cands"])
    np.testing.assert_allclose(got, g["costs"], rtol=1e-10)


def _replay(g, precision, scorer):
    pr, p, st = G.problem(g), int(g["p"]), G.settings(g)
    draws = [O.draws(st, k, p, pr.m) for k in range(1, st.generations)]
    settings = P.EmpcSettings(num_sims=st.num_sims, num_parents=st.num_parents, generations=st.generations,
                              seed=st.seed, precision=precision, scorer=scorer)
    return P.solve_empc(G.spec(g), _sched(g), settings, g["x0"], draws=draws, init_candidates=g["tap_init"])


@pytest.mark.parametrize("name", ["spec2_g3", "c1_g10", "c2_g3"])
def test_condensed_solve_fp64_replays_reference(name):
    """The reference's algorithm end to end: FP64 condensed scoring + the
    reference's random tensors reproduce its population bit for bit."""
    g = G.load("solve_" + name)
    res = _replay(g, "fp64", "condensed")
    np.testing.assert_array_equal(res.population.candidates, g["pop_cands"])
    np.testing.assert_allclose(res.population.costs, g["pop_costs"], rtol=RTOL64)
    np.testing.assert_array_equal(res.best, g["best"])
    assert res.best_cost == pytest.approx(float(g["best_cost"]), rel=RTOL64)


def test_condensed_matches_rollout_solve_fp64():
    """Same draws, same population: the scorers are the same function."""
    g = G.load("solve_c2_g3")
    a = _replay(g, "fp64", "condensed")
    b = _replay(g, "fp64", "rollout")
    np.testing.assert_array_equal(a.population.candidates, b.population.candidates)
    np.testing.assert_allclose(a.population.costs, b.population.costs, rtol=1e-10)


def test_condensed_own_rng_converges():
    """SPEC.md:665-style quality: the condensed solve reaches the same cost
    region as the rollout solve (same RNG stream; the FP32 rollout and FP64
    condensed costs differ at 1e-7, so near-ties may pick different elites)."""
    g = G.load("score_c2")
    spec, sched = G.spec(g), _sched(g)
    st_c = P.EmpcSettings(num_sims=1024, num_parents=64, generations=10, seed=1, scorer="condensed")
    st_r = P.EmpcSettings(num_sims=1024, num_parents=64, generations=10, seed=1)
    rc = P.solve_empc(spec, sched, st_c, g["x0"])
    rr = P.solve_empc(spec, sched, st_r, g["x0"])
    assert rc.best_cost == pytest.approx(rr.best_cost, rel=0.05)
    # warm start keeps working on the device-resident population
    w = P.solve_empc(spec, sched, st_c, g["x0"], prev=rc.population)
    assert w.best_cost <= rc.best_cost * (1 + 1e-6)


def test_condensed_batch_equals_single():
    """Tiling-independent sums: instance 0 of a batch reproduces the single
    solve bit for bit (per-instance RNG streams start at instance 0)."""
    g = G.load("score_c2")
    spec, sched = G.spec(g), _sched(g)
    st = P.EmpcSettings(num_sims=512, num_parents=32, generations=4, seed=3, scorer="condensed")
    single = P.solve_empc(spec, sched, st, g["x0"])
    batch = P.EmpcBatch([spec, spec, spec], sched, st).solve(np.stack([g["x0"]] * 3))
    np.testing.assert_array_equal(batch.best[0], single.best)
    assert batch.best_cost[0] == single.best_cost


@pytest.mark.parametrize("world", [2, 3])
def test_condensed_sharded_equals_unsharded(world):
    g = G.load("score_c2")
    spec, sched = G.spec(g), _sched(g)
    st = P.EmpcSettings(num_sims=512, num_parents=32, generations=4, seed=5, scorer="condensed")
    ref = P.solve_empc(spec, sched, st, g["x0"])
    (u, best, cost, row), _ = SH.solve_population_emulated(spec, sched, st, g["x0"], world)
    np.testing.assert_array_equal(best, ref.best)
    np.testing.assert_array_equal(u, ref.u)
    assert cost == ref.best_cost
