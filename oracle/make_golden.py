"""Generate the golden fixtures under tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    python oracle/make_golden.py

It imports ``knotmpc`` from /root/reference/pkg/src (read-only) and records
inputs and outputs of the hot-path functions so that (a) the oracle
restatement in ``oracle/empc_oracle.py`` can be pinned against the reference
on any machine, and (b) the GPU parity tests have reference vectors without
needing /root/reference at run time.  The fixtures are small (.npz).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _import_ref():
    sys.path.insert(0, REF)
    import knotmpc  # noqa: F401
    from knotmpc import condense, dynamics, empc, param
    return condense, dynamics, empc, param


def spec_arrays(spec, prefix=""):
    m = spec.model
    return {
        prefix + "Ad": m.Ad, prefix + "Bd": m.Bd, prefix + "wd": m.wd, prefix + "T": np.int64(spec.T),
        prefix + "Q": spec.Q, prefix + "R": spec.R, prefix + "x_goal": spec.x_goal,
        prefix + "u_goal": spec.u_goal, prefix + "u_min": spec.u_min, prefix + "u_max": spec.u_max,
    }


def main():
    condense, dynamics, empc, param = _import_ref()
    os.makedirs(OUT, exist_ok=True)

    # -- knot schedules: W for every config's (T, p) plus the reference's frozen cases
    wcases = [(5, 3), (7, 7), (8, 1), (20, 2), (20, 3), (50, 3), (50, 4), (200, 5), (23, 6), (15, 4), (11, 4),
              (120, 7), (100, 34), (99, 50)]
    wd = {}
    for T, p in wcases:
        s = param.KnotSchedule(T=T, p=p)
        wd[f"W_{T}_{p}"] = param.interpolation_matrix(s)
        co = np.array([s.coeffs(k) for k in range(T)], dtype=object)
        wd[f"idx_{T}_{p}"] = np.array([[int(a), int(b)] for a, b, _ in co], np.int64)
        wd[f"c_{T}_{p}"] = np.array([float(c) for _, _, c in co])
    np.savez_compressed(os.path.join(OUT, "knots.npz"), **wd)

    # -- the reference test system (TST/test_empc.py:20-36)
    Ad = np.array([[1.0, 0.02], [-0.4, 0.97]])
    Bd = np.array([[0.0], [0.05]])
    model = dynamics.DiscreteLinearModel(Ad, Bd, np.zeros(2), 0.02)
    spec2 = condense.MpcSpec(model, 20, Q=np.diag([10.0, 0.1]), R=0.01 * np.eye(1),
                             x_goal=np.array([0.5, 0.0]), u_goal=np.zeros(1),
                             u_min=-np.array([4.0]), u_max=np.array([4.0]))
    x02 = np.array([-0.3, 0.1])
    sched2 = param.KnotSchedule(T=20, p=3)

    # -- n-link systems built with the reference's own recipe
    def nlink_case(D, T, p, seed):
        plant = dynamics.NLinkArm(dynamics.NLinkParams(links=D))
        rng = np.random.default_rng(seed)
        q0 = rng.uniform(-np.pi, np.pi, D)
        qg = rng.uniform(-np.pi, np.pi, D)
        x0 = np.concatenate([q0, np.zeros(D)])
        xg = np.concatenate([qg, np.zeros(D)])
        mdl = dynamics.discretize(dynamics.linearize(plant.ode, x0, np.zeros(D)), 0.01)
        spec = condense.MpcSpec(mdl, T, Q=np.diag([10.0] * D + [0.1] * D), R=0.01 * np.eye(D),
                                x_goal=xg, u_goal=np.zeros(D), u_min=np.full(D, -2.0), u_max=np.full(D, 2.0))
        return spec, param.KnotSchedule(T=T, p=p), x0

    cases = {
        "spec2": (spec2, sched2, x02),
        "c1": nlink_case(2, 20, 2, 0),
        "c2": nlink_case(6, 50, 3, 0),
        "c3s": nlink_case(24, 50, 4, 0),   # C3 system, scored on a small population
    }
    # dense-Q / dense-R / drift variant of the 6-DoF system
    s6, sc6, x6 = cases["c2"]
    rng = np.random.default_rng(42)
    Mq = rng.normal(size=(12, 12))
    Mr = rng.normal(size=(6, 6))
    dense = condense.MpcSpec(dynamics.DiscreteLinearModel(s6.model.Ad, s6.model.Bd, 0.01 * rng.normal(size=12), 0.01),
                             50, Q=Mq @ Mq.T / 12, R=Mr @ Mr.T / 6 + 0.1 * np.eye(6), x_goal=s6.x_goal,
                             u_goal=0.1 * rng.normal(size=6), u_min=s6.u_min, u_max=s6.u_max)
    cases["dense"] = (dense, sc6, x6)

    for name, (spec, sched, x0) in cases.items():
        rng = np.random.default_rng(123)
        N = 64
        cands = rng.uniform(spec.u_min, spec.u_max, size=(N, sched.p, spec.model.m))
        cm = empc._CostModel(spec, sched, x0)
        d = spec_arrays(spec)
        d.update(p=np.int64(sched.p), x0=x0, cands=cands, cost_condensed=cm(cands),
                 cost_rollout=empc._rollout_costs(cands, spec, sched, x0),
                 cost_single=np.array([empc.evaluate_cost(cands[i], spec, sched, x0) for i in range(4)]))
        np.savez_compressed(os.path.join(OUT, f"score_{name}.npz"), **d)

    # -- full solves (cold and warm) plus the RNG tap for the test system and C1
    solves = {
        "spec2_g3": (cases["spec2"], empc.EmpcSettings(num_sims=64, num_parents=8, seed=7, generations=3)),
        "spec2_p1": ((spec2, param.KnotSchedule(T=20, p=1), x02), empc.EmpcSettings(num_sims=64, num_parents=8, seed=7, generations=2)),
        "spec2_kn": (cases["spec2"], empc.EmpcSettings(num_sims=8, num_parents=8, seed=7, generations=2)),
        "c1_g10": (cases["c1"], empc.EmpcSettings(num_sims=100, num_parents=6, seed=1, generations=10)),
        "c2_g3": (cases["c2"], empc.EmpcSettings(num_sims=1024, num_parents=64, seed=1, generations=3)),
    }
    for name, ((spec, sched, x0), st) in solves.items():
        res = empc.solve_empc(spec, sched, st, x0)
        warm = empc.solve_empc(spec, sched, st, x0 + 0.01, prev=res.population)
        d = spec_arrays(spec)
        d.update(p=np.int64(sched.p), x0=x0, N=np.int64(st.num_sims), K=np.int64(st.num_parents),
                 G=np.int64(st.generations), seed=np.int64(st.seed),
                 u=res.u, best=res.best, best_cost=np.float64(res.best_cost),
                 pop_cands=res.population.candidates, pop_costs=res.population.costs,
                 pop_gen=np.int64(res.population.generation),
                 warm_best=warm.best, warm_best_cost=np.float64(warm.best_cost),
                 warm_pop_cands=warm.population.candidates, warm_pop_costs=warm.population.costs,
                 warm_gen=np.int64(warm.population.generation))
        # RNG tap for generation 1 (the first evolve), in the reference's own draw order
        if st.num_sims > st.num_parents:
            g = empc._rng(st.seed, 1)
            nc = st.num_sims - st.num_parents
            d.update(tap_parents=g.integers(0, st.num_parents, size=(nc, 2)),
                     tap_take_second=g.random((nc, sched.p, spec.model.m)) < st.crossover_prob,
                     tap_mutate=g.random((nc, sched.p, spec.model.m)) < st.mutation_prob,
                     tap_noise=g.normal(size=(nc, sched.p, spec.model.m)))
            g0 = empc._rng(st.seed, 0)
            d.update(tap_init=g0.uniform(spec.u_min, spec.u_max, size=(st.num_sims, sched.p, spec.model.m)),
                     sigma=empc._mutation_sigma(spec, st, x0))
        np.savez_compressed(os.path.join(OUT, f"solve_{name}.npz"), **d)

    # -- state-bounded spec (rollout scoring path, K/empc.py:138)
    sb = condense.MpcSpec(spec2.model, 20, spec2.Q, spec2.R, spec2.x_goal, spec2.u_goal, spec2.u_min, spec2.u_max,
                          x_min=-10.0 * np.ones(2), x_max=10.0 * np.ones(2))
    pop = empc.init_population(sb, sched2, empc.EmpcSettings(num_sims=64, num_parents=8, seed=7), x02)
    np.savez_compressed(os.path.join(OUT, "bounded.npz"), cands=pop.candidates, costs=pop.costs)

    print("wrote", sorted(os.listdir(OUT)))


def closed_loop():
    """Closed-loop EMPC traces (K/closedloop.py:59-133) for the f1 parity
    test: the pendulum smoke case of TST/test_closedloop.py:234-245, the same
    with gravity (the relinearization matters), and a 2-link arm."""
    sys.path.insert(0, REF)
    from knotmpc import closedloop as cl, condense, dynamics

    def template(plant, T, umax):
        clin = dynamics.linearize(plant.ode, np.zeros(plant.n), np.zeros(plant.m))
        nj = plant.m
        return condense.MpcSpec(dynamics.discretize(clin, 0.01), T, Q=np.diag([10.0] * nj + [0.1] * nj),
                                R=0.01 * np.eye(nj), x_goal=np.zeros(plant.n), u_goal=np.zeros(nj),
                                u_min=-umax * np.ones(nj), u_max=umax * np.ones(nj))

    cases = {
        "pend0": (dynamics.Pendulum(dynamics.PendulumParams(gravity=0.0)), 30, 25.0, 3, [0.4, 0.0],
                  dict(num_sims=64, num_parents=8, generations=2), 0.5),
        "pendg": (dynamics.Pendulum(dynamics.PendulumParams()), 30, 25.0, 3, [0.8, 0.0],
                  dict(num_sims=128, num_parents=16, generations=3, seed=5), 0.3),
        "arm2": (dynamics.NLinkArm(dynamics.NLinkParams(links=2)), 20, 2.0, 3, [0.5, -0.3, 0.0, 0.0],
                 dict(num_sims=256, num_parents=16, generations=3, seed=2), 0.2),
    }
    for name, (plant, T, umax, p, goal, st, dur) in cases.items():
        tpl = template(plant, T, umax)
        ctl = cl.Controller("empc", p=p, empc=cl.EmpcSettings(**st))
        res = cl.run_closed_loop(plant, ctl, tpl, x0=np.zeros(plant.n), x_goal=np.array(goal), duration=dur,
                                 rate=100.0)
        np.savez_compressed(os.path.join(OUT, f"closedloop_{name}.npz"), states=res.states, inputs=res.inputs,
                            goal=np.array(goal), T=np.int64(T), umax=umax, p=np.int64(p), duration=dur,
                            **{"st_" + k: v for k, v in st.items()})
    print("wrote closed-loop fixtures")


def harness():
    """Rows of the reference harness (K/bench.py) for small EMPC configs, timing
    columns masked: the f4 parity fixtures."""
    sys.path.insert(0, REF)
    from knotmpc import bench as B

    cl = B.ExperimentConfig(experiment="closedloop_comparison", robot="nlink", links=(1, 2), T=20,
                            controllers=("empc:3:1", "empc:3:2"), trials=2, duration=0.2, rate=100.0, seed=7,
                            empc_sims=64, empc_parents=8, out="x.csv")
    st = B.ExperimentConfig(experiment="solve_time_scaling", robot="nlink", links=(1, 3), T=20,
                            controllers=("empc:3:2",), trials=2, rate=100.0, seed=11, empc_sims=64, empc_parents=8,
                            out="y.csv")
    pe = B.ExperimentConfig(experiment="closedloop_comparison", robot="pendulum", T=20,
                            controllers=("empc:2:2",), trials=2, duration=0.2, rate=100.0, seed=3, empc_sims=64,
                            empc_parents=8, out="z.csv")
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        for name, cfg in (("closedloop", cl), ("solvetime", st), ("pendulum", pe)):
            rows = B.run_experiment(cfg, d, workers=1)
            with open(os.path.join(OUT, f"harness_{name}.csv"), "w") as fh:
                fh.write(B.rows_to_csv_text(rows, include_timing=False))
    print("wrote harness fixtures")


def _digest(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def headline():
    """Whole solves of the benchmark configs from the real reference
    (K/empc.py:211-236) on the §8(d) systems: C3 (N=4096, K=256, G=10, cold +
    warm), C4 at G=3 and two C5 instances.  Populations are large, so the
    fixture keeps their SHA-256 (bit-identity checks), the costs, the elite
    block of C3 and the best candidate; the draws are regenerated by the
    oracle's RNG tap, which tests/test_oracle_golden.py pins to these files."""
    condense, dynamics, empc, param = _import_ref()

    def nlink_case(D, T, seed):
        plant = dynamics.NLinkArm(dynamics.NLinkParams(links=D))
        rng = np.random.default_rng(seed)
        q0 = rng.uniform(-np.pi, np.pi, D)
        qg = rng.uniform(-np.pi, np.pi, D)
        x0 = np.concatenate([q0, np.zeros(D)])
        xg = np.concatenate([qg, np.zeros(D)])
        mdl = dynamics.discretize(dynamics.linearize(plant.ode, x0, np.zeros(D)), 0.01)
        spec = condense.MpcSpec(mdl, T, Q=np.diag([10.0] * D + [0.1] * D), R=0.01 * np.eye(D),
                                x_goal=xg, u_goal=np.zeros(D), u_min=np.full(D, -2.0), u_max=np.full(D, 2.0))
        return spec, x0

    cases = {
        # name: (dof, T, p, N, K, G, system seeds, warm)
        "c3_g10": (24, 50, 4, 4096, 256, 10, [0], True),
        "c4_g3": (48, 200, 5, 16384, 1024, 3, [0], False),
        "c5_i2": (12, 50, 3, 512, 32, 10, [0, 1], False),
    }
    for name, (D, T, p, N, K, G, seeds, warm) in cases.items():
        st = empc.EmpcSettings(num_sims=N, num_parents=K, generations=G, seed=1)
        sched = param.KnotSchedule(T=T, p=p)
        d = dict(dof=np.int64(D), T=np.int64(T), p=np.int64(p), N=np.int64(N), K=np.int64(K), G=np.int64(G),
                 seed=np.int64(1), seeds=np.array(seeds, np.int64))
        for i, s in enumerate(seeds):
            spec, x0 = nlink_case(D, T, s)
            res = empc.solve_empc(spec, sched, st, x0)
            pre = f"i{i}_"
            d.update({pre + k: v for k, v in spec_arrays(spec).items()})
            d.update({pre + "x0": x0, pre + "u": res.u, pre + "best": res.best,
                      pre + "best_cost": np.float64(res.best_cost), pre + "pop_costs": res.population.costs,
                      pre + "pop_sha": np.array(_digest(res.population.candidates)),
                      pre + "pop_gen": np.int64(res.population.generation),
                      pre + "sigma": empc._mutation_sigma(spec, st, x0)})
            if name == "c3_g10":
                d[pre + "pop_elites"] = res.population.candidates[:K]
            if warm:
                wr = empc.solve_empc(spec, sched, st, x0 + 0.01, prev=res.population)
                d.update({pre + "warm_best": wr.best, pre + "warm_best_cost": np.float64(wr.best_cost),
                          pre + "warm_pop_costs": wr.population.costs,
                          pre + "warm_pop_sha": np.array(_digest(wr.population.candidates)),
                          pre + "warm_gen": np.int64(wr.population.generation)})
        np.savez_compressed(os.path.join(OUT, f"solve_{name}.npz"), **d)
        print("wrote", name)


if __name__ == "__main__":
    if sys.argv[1:] == ["closedloop"]:
        closed_loop()
    elif sys.argv[1:] == ["harness"]:
        harness()
    elif sys.argv[1:] == ["headline"]:
        headline()
    else:
        main()
        closed_loop()
        harness()
        headline()
