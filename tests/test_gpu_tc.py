"""GPU parity of the tensor-core rollout (rollout_tc_kernel: tcgen05 TF32
split precision, FP32 populations, diagonal Q) against the oracle and the
reference's golden vectors, through the C ABI.

Tolerance: the same FP32 contract as the FFMA rollout, |d|/|J| <= 1e-5
(SURVEY.md §8c P1).  Whole solves driven by the reference's random tensors
must return the reference's elites / input (P4/P5, gap-aware like
test_gpu_parity.test_solve_fp32_replays_reference).
"""

import numpy as np
import pytest

import paper_2001_04931_b200 as P
from oracle import empc_oracle as O
from tests import golden as G

pytestmark = pytest.mark.gpu

RTOL32 = 1e-5


def _sched(g):
    return P.KnotSchedule(int(g["T"]), int(g["p"]))


def _uses_tc(ctx):
    return "tcgen05" in ctx.h.describe()


@pytest.mark.parametrize("name", ["spec2", "c1", "c2", "c3s"])
def test_tc_scorer_matches_reference(name):
    g = G.load("score_" + name)
    cm = P.CostModel(G.spec(g), _sched(g), g["x0"], tensor_cores="on")
    got = cm(g["cands"])
    np.testing.assert_allclose(got, g["cost_condensed"], rtol=RTOL32)
    np.testing.assert_allclose(got, g["cost_rollout"], rtol=RTOL32)
    pr = G.problem(g)
    ctx = P.empc._context(pr.n, pr.m, pr.T, int(g["p"]), 1, 1, 1, False, "fp32")
    assert _uses_tc(ctx), ctx.h.describe()


def test_tc_dense_q_falls_back():
    """Dense Q is not a tensor-core shape: the FFMA rollout scores it."""
    g = G.load("score_dense")
    got = P.CostModel(G.spec(g), _sched(g), g["x0"], tensor_cores="on")(g["cands"])
    np.testing.assert_allclose(got, g["cost_rollout"], rtol=RTOL32)


@pytest.mark.parametrize("num", [1, 3, 127, 128, 129, 1000])
def test_tc_ragged_batches(num):
    """Partial and multiple 128-candidate tiles."""
    g = G.load("score_c2")
    pr = G.problem(g)
    rng = np.random.default_rng(num)
    cands = rng.uniform(pr.u_min, pr.u_max, size=(num, int(g["p"]), pr.m))
    got = P.CostModel(G.spec(g), _sched(g), g["x0"], tensor_cores="on")(cands)
    np.testing.assert_allclose(got, O.rollout_costs(cands, pr, g["x0"]), rtol=RTOL32)


@pytest.mark.parametrize("dof,T,p", [(1, 20, 1), (3, 30, 2), (5, 25, 3), (12, 50, 3), (24, 50, 4), (32, 40, 3),
                                     (48, 200, 5), (40, 30, 2)])
def test_tc_every_state_size(dof, T, p):
    """Every padded state size (n = 2 dof) against the FP64 oracle rollout on
    the reference's synthetic N-link arms."""
    from paper_2001_04931_b200 import workloads as W

    spec, x0 = W.nlink_problem(dof, T, 0)
    pr = O.Problem.from_spec(spec)
    rng = np.random.default_rng(dof)
    cands = rng.uniform(pr.u_min, pr.u_max, size=(300, p, pr.m))
    sched = P.KnotSchedule(T, p)
    got = P.CostModel(spec, sched, x0, tensor_cores="on")(cands)
    np.testing.assert_allclose(got, O.rollout_costs(cands, pr, x0), rtol=RTOL32)
    ffma = P.CostModel(spec, sched, x0, tensor_cores="off")(cands)
    np.testing.assert_allclose(got, ffma, rtol=RTOL32)


def test_tc_dense_r():
    from paper_2001_04931_b200 import workloads as W

    spec, x0 = W.nlink_problem(6, 30, 1)
    m = spec.R.shape[0]
    R = 0.01 * np.eye(m) + 0.002 * (np.ones((m, m)) - np.eye(m))
    spec = P.MpcSpec(spec.model, spec.T, Q=spec.Q, R=R, x_goal=spec.x_goal, u_goal=0.1 * np.ones(m),
                     u_min=spec.u_min, u_max=spec.u_max)
    pr = O.Problem.from_spec(spec)
    cands = np.random.default_rng(5).uniform(pr.u_min, pr.u_max, size=(200, 3, m))
    got = P.CostModel(spec, P.KnotSchedule(30, 3), x0, tensor_cores="on")(cands)
    np.testing.assert_allclose(got, O.rollout_costs(cands, pr, x0), rtol=RTOL32)


@pytest.mark.parametrize("name", ["spec2_g3", "c1_g10", "c2_g3"])
def test_tc_solve_replays_reference(name):
    g = G.load("solve_" + name)
    pr, p, st = G.problem(g), int(g["p"]), G.settings(g)
    init, trace = O.solve_trace(pr, p, st, g["x0"])
    gaps = []
    for pop, _ in trace[:-1]:
        c = np.sort(pop.costs)
        K = st.num_parents
        rel = np.abs(np.diff(c[:min(K + 1, c.size)])) / np.abs(c[:min(K, c.size - 1)])
        distinct = rel[rel > 0]
        gaps.append(distinct.min() if distinct.size else np.inf)
    draws = [O.draws(st, k, p, pr.m) for k in range(1, st.generations)]
    settings = P.EmpcSettings(num_sims=st.num_sims, num_parents=st.num_parents, generations=st.generations,
                              seed=st.seed, tensor_cores="on")
    res = P.solve_empc(G.spec(g), _sched(g), settings, g["x0"], draws=draws, init_candidates=g["tap_init"])
    if min(gaps) > 1e-4:
        np.testing.assert_allclose(res.best, g["best"], rtol=1e-5, atol=1e-6)
        assert res.best_cost == pytest.approx(float(g["best_cost"]), rel=RTOL32)
    else:
        assert res.best_cost == pytest.approx(float(g["best_cost"]), rel=1e-4)


def test_tc_production_solve_costs_match_oracle():
    """In-kernel Philox breeding + tensor-core scoring: every population cost
    agrees with the FP64 oracle rollout of the returned candidates."""
    from paper_2001_04931_b200 import workloads as W

    spec, x0 = W.nlink_problem(24, 50, 0)
    st = P.EmpcSettings(num_sims=1024, num_parents=64, generations=4, seed=1, tensor_cores="on")
    res = P.solve_empc(spec, P.KnotSchedule(50, 4), st, x0)
    pr = O.Problem.from_spec(spec)
    np.testing.assert_allclose(res.population.costs, O.rollout_costs(res.population.candidates, pr, x0),
                               rtol=RTOL32)
    assert res.best_cost == pytest.approx(float(np.min(res.population.costs)))
    np.testing.assert_array_equal(np.sort(res.population.costs[:64]), res.population.costs[:64])


def test_tc_batched_instances_match_oracle():
    from paper_2001_04931_b200 import workloads as W

    w = W.Workload("mini", 12, 50, 3, 512, 32, 3, instances=6)
    specs, x0s = W.build(w)
    batch = P.EmpcBatch(specs, w.schedule(), w.settings(tensor_cores="on"))
    assert _uses_tc(batch.ctx), batch.ctx.h.describe()
    r = batch.solve(x0s)
    for i in (0, 5):
        pr = O.Problem.from_spec(specs[i])
        np.testing.assert_allclose(r.population.costs[i], O.rollout_costs(r.population.candidates[i], pr, x0s[i]),
                                   rtol=RTOL32)


def test_tc_init_generation_equals_ffma_population():
    """Same Philox draws, different scoring machine: the cold-start
    populations are identical and the costs agree to the FP32 contract."""
    from paper_2001_04931_b200 import workloads as W

    spec, x0 = W.nlink_problem(48, 200, 0)
    sched = P.KnotSchedule(200, 5)
    a = P.solve_empc(spec, sched, P.EmpcSettings(num_sims=2048, num_parents=128, generations=1, seed=2,
                                                 tensor_cores="on"), x0)
    b = P.solve_empc(spec, sched, P.EmpcSettings(num_sims=2048, num_parents=128, generations=1, seed=2,
                                                 tensor_cores="off"), x0)
    np.testing.assert_array_equal(a.population.candidates, b.population.candidates)
    np.testing.assert_allclose(a.population.costs, b.population.costs, rtol=RTOL32)


def test_tc_multi_tile_ctas_match_ffma_and_oracle():
    """>= 4 x 148 instances with several tiles each: one CTA per instance
    loops over its tiles (problem staged once).  Cold start = same Philox
    population as the FFMA kernel, costs to the FP32 contract; a 3-generation
    solve's population costs match the oracle."""
    from paper_2001_04931_b200 import workloads as W

    w = W.Workload("multi", 3, 20, 2, 300, 20, 1, instances=600)
    specs, x0s = W.build(w)
    on = P.EmpcBatch(specs, w.schedule(), w.settings(tensor_cores="on"))
    assert _uses_tc(on.ctx), on.ctx.h.describe()
    off = P.EmpcBatch(specs, w.schedule(), w.settings(tensor_cores="off"))
    a, b = on.solve(x0s), off.solve(x0s)
    np.testing.assert_array_equal(a.population.candidates, b.population.candidates)
    np.testing.assert_allclose(a.population.costs, b.population.costs, rtol=RTOL32)
    w3 = W.Workload("multi", 3, 20, 2, 300, 20, 3, instances=600)
    r = P.EmpcBatch(specs, w3.schedule(), w3.settings(tensor_cores="on")).solve(x0s)
    for i in (0, 311, 599):
        pr = O.Problem.from_spec(specs[i])
        np.testing.assert_allclose(r.population.costs[i], O.rollout_costs(r.population.candidates[i], pr, x0s[i]),
                                   rtol=RTOL32)


def test_tc_population_sharding_matches_unsharded():
    """C4-style population sharding with the tensor-core rollout on every rank
    (2 ranks in lock-step on one GPU): the unsharded result bit for bit, since
    a candidate's arithmetic does not depend on its tile or row."""
    from paper_2001_04931_b200 import workloads as W
    from paper_2001_04931_b200.shard import solve_population_emulated

    spec, x0 = W.nlink_problem(32, 30, 0)
    sched = P.KnotSchedule(30, 3)
    st = P.EmpcSettings(num_sims=5824, num_parents=1024, generations=3, seed=5)
    ref = P.solve_empc(spec, sched, st, x0)
    ctx = P.empc._context(64, 32, 30, 3, 5824, 1024, 1, False, "fp32")
    assert _uses_tc(ctx), ctx.h.describe()
    (u, best, cost, row), shards = solve_population_emulated(spec, sched, st, x0, 2)
    np.testing.assert_array_equal(best, ref.best)
    np.testing.assert_array_equal(u, ref.u)
    assert cost == ref.best_cost
