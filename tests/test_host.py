"""Host-side logic of the drop-in package (no GPU): problem types and their
validation, knot schedules, sigma schedule, synthetic workloads, and the
RNG contract model.  Mirrors TST/test_param.py, TST/test_empc.py:146-156 and
TST/test_condense.py validation cases."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import empc as E
from paper_2001_04931_b200 import workloads as W
from oracle import empc_oracle as O
from tests import golden as G
from tests.philox_model import breed_draws, philox

W_T5_P3 = np.array([[1.0, 0, 0], [0.5, 0.5, 0], [0, 1.0, 0], [0, 0.5, 0.5], [0, 0, 1.0]])


# ---- knot schedules (TST/test_param.py)

def test_knot_spacing_values():
    assert P.knot_spacing(50, 5) == pytest.approx(12.25)
    assert P.knot_spacing(5, 3) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        P.knot_spacing(10, 1)
    with pytest.raises(ValueError):
        P.knot_spacing(5, 6)


def test_interp_coeffs_and_snap():
    assert P.interp_coeffs(3, 2.0)[:2] == (1, 2)
    assert P.interp_coeffs(0, 2.0) == (0, 0, 0.0)
    assert P.interp_coeffs(2, 1.00000000005) == (2, 2, 0.0)


def test_schedule_validation():
    for T, p in ((10, 0), (10, 11), (0, 1)):
        with pytest.raises(ValueError):
            P.KnotSchedule(T=T, p=p)
    s = P.KnotSchedule(T=10, p=4)
    with pytest.raises(ValueError):
        s.coeffs(10)
    assert P.KnotSchedule(8, 1).spacing is None


def test_interpolation_matrix_matches_reference_goldens():
    g = G.load("knots")
    np.testing.assert_allclose(P.interpolation_matrix(P.KnotSchedule(5, 3)), W_T5_P3, atol=1e-12)
    for key in g:
        if key.startswith("W_"):
            _, T, p = key.split("_")
            np.testing.assert_array_equal(P.interpolation_matrix(P.KnotSchedule(int(T), int(p))), g[key])
            i1, i2, c = P.param.schedule_arrays(int(T), int(p))
            np.testing.assert_array_equal(np.stack([i1, i2], 1), g[f"idx_{T}_{p}"])
            np.testing.assert_array_equal(c, g[f"c_{T}_{p}"])


@settings(max_examples=60, deadline=None)
@given(st.integers(2, 120).flatmap(lambda T: st.tuples(st.just(T), st.integers(1, T))))
def test_interpolation_matrix_invariants(Tp):
    T, p = Tp
    W_ = P.interpolation_matrix(P.KnotSchedule(T=T, p=p))
    assert W_.shape == (T, p) and np.all(W_ >= 0)
    np.testing.assert_allclose(W_.sum(axis=1), 1.0, atol=1e-12)
    assert np.max(np.count_nonzero(W_, axis=1)) <= 2
    np.testing.assert_allclose(W_, O.interpolation_matrix(T, p), atol=0)


def test_input_at_and_trajectory_validation():
    sched = P.KnotSchedule(T=23, p=6)
    U = np.random.default_rng(5).normal(size=(6, 2))
    traj = P.KnotTrajectory(U, sched)
    full = P.interpolation_matrix(sched) @ U
    for k in range(23):
        np.testing.assert_allclose(P.input_at(traj, k), full[k], atol=1e-14)
    with pytest.raises(ValueError):
        P.KnotTrajectory(np.zeros((4, 1)), P.KnotSchedule(10, 3))


# ---- settings / spec validation (TST/test_empc.py:146-156, K/condense.py:57-81)

def test_settings_validation():
    for kw in (dict(num_sims=0), dict(num_parents=100, num_sims=50), dict(generations=0), dict(mutation_prob=1.5),
               dict(crossover_prob=-0.1), dict(precision="fp16")):
        with pytest.raises(ValueError):
            P.EmpcSettings(**kw)
    assert P.EmpcSettings(num_sims=8, num_parents=8).num_parents == 8


def _model():
    return P.DiscreteLinearModel(np.array([[1.0, 0.02], [-0.4, 0.97]]), np.array([[0.0], [0.05]]), np.zeros(2), 0.02)


def test_spec_validation_and_broadcasting():
    mdl = _model()
    s = P.MpcSpec(mdl, 20, np.diag([10.0, 0.1]), 0.01 * np.eye(1), 0.5, 0.0, -4.0, 4.0)
    assert s.x_goal.shape == (2,) and s.u_min.shape == (1,)
    assert not s.has_state_bounds
    assert P.MpcSpec(mdl, 20, np.eye(2), np.eye(1), 0, 0, -1, 1, x_min=-10.0).has_state_bounds
    bad = [dict(T=0), dict(Q=np.eye(3)), dict(Q=np.array([[1.0, 1.0], [0.0, 1.0]])), dict(Q=-np.eye(2)),
           dict(R=np.zeros((1, 1))), dict(u_min=5.0)]
    for kw in bad:
        args = dict(model=mdl, T=20, Q=np.eye(2), R=np.eye(1), x_goal=0.0, u_goal=0.0, u_min=-4.0, u_max=4.0)
        args.update(kw)
        with pytest.raises(ValueError):
            P.MpcSpec(**args)


def test_mutation_sigma_matches_oracle():
    g = G.load("solve_c1_g10")
    spec = G.spec(g)
    for st_ in (P.EmpcSettings(seed=1), P.EmpcSettings(sigma_noise=np.array([0.3, 0.7]), dist_ref=0.5)):
        want = O.mutation_sigma(O.Problem.from_spec(spec), O.Settings.from_settings(st_), g["x0"])
        np.testing.assert_array_equal(E._mutation_sigma(spec, st_, g["x0"]), want)
    np.testing.assert_array_equal(E._mutation_sigma(spec, P.EmpcSettings(seed=1), g["x0"]), g["sigma"])


def test_diagonal_q_detection_matches_reference_rule():
    assert E._is_diag(np.diag([1.0, 2.0]))
    assert not E._is_diag(np.array([[1.0, 0.1], [0.1, 1.0]]))


def test_batch_sigma_matches_single():
    w = W.Workload("mini", 2, 20, 2, 16, 4, 2, instances=3)
    specs, x0s = W.build(w)
    st_ = w.settings()
    b = P.EmpcBatch.__new__(P.EmpcBatch)
    b.probs = E.stack_specs(specs)
    b.I, b.n, b.m, b.settings = 3, 4, 2, st_
    for i in range(3):
        np.testing.assert_allclose(b.sigma(x0s)[i], E._mutation_sigma(specs[i], st_, x0s[i]), rtol=1e-15)


# ---- synthetic workloads: the reference recipe reproduces the reference systems

@pytest.mark.parametrize("name,dof,T", [("c1", 2, 20), ("c2", 6, 50), ("c3s", 24, 50)])
def test_workload_systems_match_reference(name, dof, T):
    g = G.load("score_" + name)
    spec, x0 = W.nlink_problem(dof, T, 0)
    np.testing.assert_allclose(x0, g["x0"], rtol=0, atol=0)
    np.testing.assert_allclose(spec.x_goal, g["x_goal"], atol=0)
    np.testing.assert_allclose(spec.model.Ad, g["Ad"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(spec.model.Bd, g["Bd"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(spec.model.wd, g["wd"], rtol=1e-6, atol=1e-12)


def test_workload_accounting():
    w = W.WORKLOADS["c3"]
    assert w.scored_per_solve == 4096 + 9 * 3840
    assert w.flop_per_candidate == 239616
    assert W.WORKLOADS["c4"].flop_per_candidate == 3732480
    assert W.WORKLOADS["c5"].scored_per_solve == (512 + 9 * 480) * 8192


# ---- RNG contract model

def test_philox_model_known_answers():
    kat = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
           ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
           ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
            (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]
    for ctr, key, want in kat:
        got = philox(*ctr, *key)
        assert tuple(int(v) for v in got) == want


def test_breed_stream_statistics():
    parents, take, mut, z = breed_draws(11, 3, 20000, 24, 64, 0.5, 0.5)
    assert parents.min() >= 0 and parents.max() < 64
    assert abs(take.mean() - 0.5) < 0.005 and abs(mut.mean() - 0.5) < 0.005
    assert abs(z.mean()) < 0.01 and abs(z.std() - 1.0) < 0.01


def test_state_bounds_need_a_finite_entry():
    """K/condense.py:83-87: all-infinite state bounds are no bounds (the
    condensed scorer stays available)."""
    import numpy as np

    import paper_2001_04931_b200 as P
    from paper_2001_04931_b200 import empc as E

    model = P.DiscreteLinearModel(np.eye(2), np.ones((2, 1)), np.zeros(2), 0.01)
    base = dict(Q=np.eye(2), R=np.eye(1), x_goal=np.zeros(2), u_goal=np.zeros(1), u_min=-np.ones(1),
                u_max=np.ones(1))
    inf = P.MpcSpec(model, 5, x_min=-np.inf * np.ones(2), x_max=np.inf * np.ones(2), **base)
    fin = P.MpcSpec(model, 5, x_min=np.array([-np.inf, -3.0]), **base)
    assert not E._has_state_bounds(inf) and E._scorer_code("condensed", inf) == 1
    assert E._has_state_bounds(fin) and E._scorer_code("condensed", fin) == 0

    class Dummy:  # duck-typed spec without the property
        x_min = np.array([-np.inf, -np.inf])
        x_max = None

    assert not E._has_state_bounds(Dummy())


def test_bench_gpus_self_launch(monkeypatch):
    """`bench.py --gpus N` without a torchrun environment starts N ranks
    itself (one process per GPU, 127.0.0.1 rendezvous) with the same args."""
    import importlib
    import sys

    import bench

    importlib.reload(bench)
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--config", "c5", "--steps", "3"])
    try:
        bench.main()
    except SystemExit as e:
        assert e.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-6:] == ["--gpus", "4", "--config", "c5", "--steps", "3"]
