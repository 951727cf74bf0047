"""Pin the CPU oracle (oracle/empc_oracle.py) against the golden vectors the
real reference produced (oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import empc_oracle as O
from tests import golden as G

SCORES = ["spec2", "c1", "c2", "c3s", "dense"]
SOLVES = ["spec2_g3", "spec2_p1", "spec2_kn", "c1_g10", "c2_g3"]


def test_interpolation_matrices_match_reference():
    g = G.load("knots")
    for key in g:
        if not key.startswith("W_"):
            continue
        _, T, p = key.split("_")
        T, p = int(T), int(p)
        W = O.interpolation_matrix(T, p)
        np.testing.assert_array_equal(W, g[key])
        i1, i2, c = O.knot_coeffs(T, p)
        np.testing.assert_array_equal(np.stack([i1, i2], 1), g[f"idx_{T}_{p}"])
        np.testing.assert_array_equal(c, g[f"c_{T}_{p}"])


@pytest.mark.parametrize("name", SCORES)
def test_scorers_match_reference(name):
    g = G.load("score_" + name)
    pr = G.problem(g)
    p = int(g["p"])
    cm = O.CostModel(pr, p, g["x0"])
    np.testing.assert_allclose(cm(g["cands"]), g["cost_condensed"], rtol=1e-12)
    np.testing.assert_allclose(O.rollout_costs(g["cands"], pr, g["x0"]), g["cost_rollout"], rtol=1e-12)
    single = [O.evaluate_cost(g["cands"][i], pr, p, g["x0"]) for i in range(4)]
    np.testing.assert_allclose(single, g["cost_single"], rtol=1e-12)
    # condensed and rollout scoring are the same function (K/empc.py:122-152)
    np.testing.assert_allclose(g["cost_condensed"], g["cost_rollout"], rtol=1e-10)


@pytest.mark.parametrize("name", SOLVES)
def test_solves_match_reference(name):
    g = G.load("solve_" + name)
    pr, p, st = G.problem(g), int(g["p"]), G.settings(g)
    res = O.solve_empc(pr, p, st, g["x0"])
    # same numpy RNG calls in the same order -> identical populations
    np.testing.assert_array_equal(res.population.candidates, g["pop_cands"])
    np.testing.assert_allclose(res.population.costs, g["pop_costs"], rtol=1e-12)
    np.testing.assert_array_equal(res.best, g["best"])
    np.testing.assert_array_equal(res.u, g["u"])
    assert res.best_cost == pytest.approx(float(g["best_cost"]), rel=1e-12)
    assert res.population.generation == int(g["pop_gen"])
    warm = O.solve_empc(pr, p, st, g["x0"] + 0.01, prev=res.population)
    np.testing.assert_array_equal(warm.population.candidates, g["warm_pop_cands"])
    assert warm.best_cost == pytest.approx(float(g["warm_best_cost"]), rel=1e-12)
    assert warm.population.generation == int(g["warm_gen"])


@pytest.mark.parametrize("name", ["spec2_g3", "c1_g10", "c2_g3"])
def test_rng_tap_matches_reference(name):
    g = G.load("solve_" + name)
    st, p, m = G.settings(g), int(g["p"]), g["Bd"].shape[1]
    d = O.draws(st, 1, p, m)
    np.testing.assert_array_equal(d.parents, g["tap_parents"])
    np.testing.assert_array_equal(d.take_second, g["tap_take_second"])
    np.testing.assert_array_equal(d.mutate, g["tap_mutate"])
    np.testing.assert_array_equal(d.noise, g["tap_noise"])
    init = O.rng(st.seed, 0).uniform(g["u_min"], g["u_max"], size=(st.num_sims, p, m))
    np.testing.assert_array_equal(init, g["tap_init"])
    np.testing.assert_array_equal(O.mutation_sigma(G.problem(g), st, g["x0"]), g["sigma"])


def test_state_bounded_rollout_path():
    g = G.load("score_spec2")
    pr = G.problem(g)
    pr.state_bounded = True
    st = O.Settings(num_sims=64, num_parents=8, seed=7)
    pop = O.init_population(pr, 3, st, g["x0"])
    b = G.load("bounded")
    np.testing.assert_array_equal(pop.candidates, b["cands"])
    np.testing.assert_allclose(pop.costs, b["costs"], rtol=1e-12)


def test_trace_replay_reproduces_solve():
    """Replaying the recorded draws through evolve_generation(d=...) gives the
    reference's solve (the injection path the GPU parity tests use)."""
    g = G.load("solve_c1_g10")
    pr, p, st = G.problem(g), int(g["p"]), G.settings(g)
    init, trace = O.solve_trace(pr, p, st, g["x0"])
    np.testing.assert_array_equal(trace[-1][0].candidates, g["pop_cands"])
    np.testing.assert_array_equal(init, g["tap_init"])


def test_qp_optimum_below_empc():
    g = G.load("solve_spec2_g3")
    pr, p = G.problem(g), int(g["p"])
    opt = O.qp_optimum(pr, p, g["x0"])
    assert opt <= float(g["best_cost"]) + 1e-9


@pytest.mark.parametrize("name", ["c3_g10", "c4_g3", "c5_i2"])
def test_headline_solves_match_reference(name):
    """The benchmark configs (BASELINE configs C3, C4 at G=3, two C5
    instances): the oracle's cold solve reproduces the real reference's
    population bit for bit (SHA-256 of the FP64 candidates)."""
    g = G.load("solve_" + name)
    for i in range(len(g["seeds"])):
        gi = G.instance(g, i)
        pr, p, st = G.problem(gi), int(gi["p"]), G.settings(gi)
        res = O.solve_empc(pr, p, st, gi["x0"])
        assert G.digest(res.population.candidates) == str(gi["pop_sha"])
        np.testing.assert_allclose(res.population.costs, gi["pop_costs"], rtol=1e-12)
        np.testing.assert_array_equal(res.best, gi["best"])
        np.testing.assert_array_equal(O.mutation_sigma(pr, st, gi["x0"]), gi["sigma"])
        if "pop_elites" in gi:
            np.testing.assert_array_equal(res.population.candidates[:st.num_parents], gi["pop_elites"])
        if "warm_pop_sha" in gi:
            warm = O.solve_empc(pr, p, st, gi["x0"] + 0.01, prev=res.population)
            assert G.digest(warm.population.candidates) == str(gi["warm_pop_sha"])
            np.testing.assert_array_equal(warm.best, gi["warm_best"])
