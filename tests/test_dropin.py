"""Drop-in boundary with the reference's OWN objects (CPU).

``paper_2001_04931_b200.solve_empc`` / ``init_population`` /
``evolve_generation`` are called with ``knotmpc.MpcSpec``,
``knotmpc.KnotSchedule``, ``knotmpc.EmpcSettings`` and ``knotmpc.Population``
instances (the signature of K/empc.py:162-236) and the arrays that cross the
C ABI are recorded by a stand-in for the native handle: they must be exactly
the ones the package's own mirror types produce.  No GPU is involved (the
compute path is covered by the -m gpu tests); the reference is imported from
/root/reference when present and the test skips otherwise (the GPU box does
not have it).
"""

import ctypes as C
import os
import sys

import numpy as np
import pytest

import paper_2001_04931_b200 as P
from paper_2001_04931_b200 import _native as nat
from paper_2001_04931_b200 import empc as E

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")


def _array_at(ptr):
    """The numpy array behind a pointer handed to the ABI (kept alive by nat._keep)."""
    addr = ptr.value if isinstance(ptr, C.c_void_p) else ptr
    io = [a for ctx in E._contexts.values() if getattr(ctx, "_io", None) for a in ctx._io.values()]
    for a in list(reversed(nat._keep)) + io:
        base = a.ctypes.data
        if base <= addr < base + max(a.nbytes, 1):  # the array or a packed part of it
            return a.reshape(-1)[(addr - base) // a.itemsize:]
    raise KeyError(addr)


class FakeHandle:
    log = []

    def __init__(self, n, m, T, p, num_sims, num_parents, instances=1, dense_q=False, precision=0, device=0):
        self.dims = nat.empc_dims(n, m, T, p, num_sims, num_parents, instances, int(bool(dense_q)), precision, device)
        self.slots = 0
        FakeHandle.log.append(("create", (n, m, T, p, num_sims, num_parents, instances, bool(dense_q), precision)))

    def set_tensor_cores(self, mode):
        FakeHandle.log.append(("tc", mode))

    def call(self, name, *args):
        d = self.dims
        if name == "empc_pop_alloc":
            args[0]._obj.value = self.slots
            self.slots += 1
        elif name == "empc_set_schedule":
            FakeHandle.log.append((name, [_array_at(a).copy() for a in args]))
        elif name == "empc_set_problems":
            FakeHandle.log.append((name, [_array_at(a).copy() for a in args[2:]]))
        elif name == "empc_pop_write":
            FakeHandle.log.append((name, _array_at(args[1]).copy(), _array_at(args[2]).copy()))
        elif name == "empc_run":
            a = args[0]._obj
            rec = {f: getattr(a, f) for f in ("init", "rescore", "evolves", "generation0", "seed", "mutation_prob",
                                              "crossover_prob")}
            rec["x0"] = _array_at(a.x0).copy()
            rec["sigma"] = _array_at(a.sigma).copy()
            FakeHandle.log.append((name, rec))
            for ptr in (a.u_out, a.best_out, a.best_cost):
                _array_at(ptr)[...] = 1.0
        else:
            FakeHandle.log.append((name, args))


@pytest.fixture
def fake(monkeypatch):
    monkeypatch.setattr(nat, "Handle", FakeHandle)
    monkeypatch.setattr(E, "_contexts", {})
    FakeHandle.log = []
    return FakeHandle


@pytest.fixture(scope="module")
def K():
    sys.path.insert(0, REF)
    import knotmpc

    return knotmpc


def _specs(K):
    rng = np.random.default_rng(0)
    Ad = np.eye(4) + 0.01 * rng.normal(size=(4, 4))
    Bd = 0.05 * rng.normal(size=(4, 2))
    wd = 0.001 * rng.normal(size=4)
    kw = dict(T=20, Q=np.diag([10.0, 10.0, 0.1, 0.1]), R=0.01 * np.eye(2), x_goal=np.array([0.5, -0.2, 0.0, 0.0]),
              u_goal=np.zeros(2), u_min=-np.ones(2), u_max=np.ones(2))
    ref = K.MpcSpec(K.DiscreteLinearModel(Ad, Bd, wd, 0.01), **kw)
    own = P.MpcSpec(P.DiscreteLinearModel(Ad, Bd, wd, 0.01), **kw)
    return ref, own


def _record(fn):
    FakeHandle.log = []
    fn()
    return list(FakeHandle.log)


def _same(la, lb):
    assert [e[0] for e in la] == [e[0] for e in lb]
    for a, b in zip(la, lb):
        if a[0] in ("empc_set_schedule", "empc_set_problems"):
            for x, y in zip(a[1], b[1]):
                np.testing.assert_array_equal(x, y)
        elif a[0] == "empc_run":
            for k in a[1]:
                np.testing.assert_array_equal(a[1][k], b[1][k])
        elif a[0] == "empc_pop_write":
            np.testing.assert_array_equal(a[1], b[1])
            np.testing.assert_array_equal(a[2], b[2])
        else:
            assert a[1] == b[1]


def test_solve_empc_accepts_reference_objects(fake, K):
    ref_spec, own_spec = _specs(K)
    x0 = np.array([-0.3, 0.1, 0.0, 0.2])
    rs = K.EmpcSettings(num_sims=128, num_parents=16, generations=3, seed=9, mutation_prob=0.3, crossover_prob=0.6,
                        sigma_scale=0.1, dist_ref=0.5)
    os_ = P.EmpcSettings(num_sims=128, num_parents=16, generations=3, seed=9, mutation_prob=0.3, crossover_prob=0.6,
                         sigma_scale=0.1, dist_ref=0.5)
    a = _record(lambda: P.solve_empc(ref_spec, K.KnotSchedule(20, 3), rs, x0))
    E._contexts.clear()
    b = _record(lambda: P.solve_empc(own_spec, P.KnotSchedule(20, 3), os_, x0))
    _same(a, b)
    run = [e for e in a if e[0] == "empc_run"][0][1]
    assert (run["init"], run["evolves"], run["generation0"], run["seed"]) == (1, 2, 1, 9)
    # sigma is the reference's own _mutation_sigma (K/empc.py:73-82)
    np.testing.assert_array_equal(run["sigma"], K.empc._mutation_sigma(ref_spec, rs, x0))
    res = P.solve_empc(ref_spec, K.KnotSchedule(20, 3), rs, x0)
    assert res.u.shape == (2,) and res.best.shape == (3, 2)


def test_warm_start_from_reference_population(fake, K):
    ref_spec, _ = _specs(K)
    rs = K.EmpcSettings(num_sims=64, num_parents=8, generations=2, seed=3)
    x0 = np.zeros(4)
    pop = K.init_population(ref_spec, K.KnotSchedule(20, 3), rs, x0)  # the reference's own (CPU) population
    log = _record(lambda: P.solve_empc(ref_spec, K.KnotSchedule(20, 3), rs, x0, prev=pop))
    w = [e for e in log if e[0] == "empc_pop_write"][0]
    np.testing.assert_array_equal(w[1].reshape(pop.candidates.shape), pop.candidates)
    np.testing.assert_array_equal(w[2].reshape(pop.costs.shape), pop.costs)
    run = [e for e in log if e[0] == "empc_run"][0][1]
    assert (run["init"], run["rescore"], run["evolves"], run["generation0"]) == (0, 1, 2, pop.generation)


def test_reference_settings_validation_is_preserved(K):
    with pytest.raises(ValueError):
        P.EmpcSettings(num_sims=4, num_parents=5)
    with pytest.raises(ValueError):
        K.EmpcSettings(num_sims=4, num_parents=5)
