"""Batched plant linearization / discretization / RK4 on the device (SURVEY
§8 f3) against the host restatement of K/dynamics.py:241-330 (which the CPU
tests pin to the reference's closed-loop traces).

Tolerances: the central differences divide rounding noise of the ODE by the
step eps = 1e-6, so device and host Jacobians agree to ~1e-10 relative of
|f|; the exponential (Taylor + squaring vs scipy's Pade) to ~1e-14.
"""

import numpy as np
import pytest

from paper_2001_04931_b200 import closedloop as CL
from paper_2001_04931_b200 import dynamics as D

PLANTS = {
    "pend0": lambda: D.Pendulum(D.PendulumParams(gravity=0.0)),
    "pendg": lambda: D.Pendulum(D.PendulumParams(mass=1.3, length=0.7)),
    "arm2": lambda: D.NLinkArm(D.NLinkParams(links=2)),
    "arm6g": lambda: D.NLinkArm(D.NLinkParams(links=6, gravity=9.81, mass=np.linspace(0.5, 1.5, 6))),
    "arm12": lambda: D.NLinkArm(D.NLinkParams(links=12)),
    "arm24": lambda: D.NLinkArm(D.NLinkParams(links=24)),
    "arm48": lambda: D.NLinkArm(D.NLinkParams(links=48)),
}


def _points(plant, count, seed):
    rng = np.random.default_rng(seed)
    L = plant.m
    xs = np.concatenate([rng.uniform(-np.pi, np.pi, (count, plant.n - L)), rng.normal(size=(count, L)) * 0.3], axis=1)
    us = rng.normal(size=(count, L))
    return xs, us


def test_device_plant_type_errors():
    with pytest.raises(TypeError):
        D.linearize_discretize(object(), np.zeros((1, 2)))
    with pytest.raises(ValueError):
        D.linearize_discretize(D.Pendulum(), np.zeros((1, 3)))
    with pytest.raises(ValueError):
        D.linearize_discretize(D.Pendulum(), np.zeros((1, 2)), method="tustin")


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(PLANTS))
@pytest.mark.parametrize("method", ["exact", "euler"])
def test_linearize_discretize_matches_host(name, method):
    plant = PLANTS[name]()
    count = 3 if plant.m >= 24 else 17
    xs, us = _points(plant, count, 7)
    Ad, Bd, wd = D.linearize_discretize(plant, xs, us, 0.01, method)
    for i in range(count):
        h = D.discretize(D.linearize(plant.ode, xs[i], us[i]), 0.01, method)
        # central-difference noise (rounding of f amplified by 1/eps and by the
        # conditioning of the inertia matrix) measured on the host itself: the
        # spread between eps = 1e-6 and 1.3e-6, x20, plus the 1e-16 |f| / eps floor
        h2 = D.discretize(D.linearize(plant.ode, xs[i], us[i], eps=1.3e-6), 0.01, method)
        f = max(1.0, np.abs(plant.ode(xs[i], us[i])).max())
        noise = max(20 * max(np.abs(h2.Ad - h.Ad).max(), np.abs(h2.Bd - h.Bd).max()),
                    100 * 1.1e-16 * f / 1e-6 * 0.01)
        np.testing.assert_allclose(Ad[i], h.Ad, rtol=1e-9, atol=noise)
        np.testing.assert_allclose(Bd[i], h.Bd, rtol=1e-9, atol=noise)
        np.testing.assert_allclose(wd[i], h.wd, rtol=1e-8, atol=noise * (1 + np.abs(xs[i]).sum() + np.abs(us[i]).sum()))


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["pend0", "pendg", "arm2", "arm6g", "arm12", "arm24"])
def test_integrate_batch_matches_host(name):
    plant = PLANTS[name]()
    xs, us = _points(plant, 9, 3)
    got = D.integrate_batch(plant, xs, us, 0.01, 10)
    for i in range(xs.shape[0]):
        want = D.integrate(plant.ode, xs[i], us[i], 0.01, substeps=10)
        np.testing.assert_allclose(got[i], want, rtol=1e-11, atol=1e-12)


@pytest.mark.gpu
def test_fleet_device_models_match_host_models():
    plants = [D.NLinkArm(D.NLinkParams(links=3)) for _ in range(5)]
    tpl = P_template(plants[0])
    goals = np.zeros((5, 6))
    ctl = CL.Controller("empc", p=3, empc=CL.EmpcSettings(num_sims=256, num_parents=16, generations=2))
    dev = CL.ClosedLoopFleet(plants, ctl, tpl, goals, rate=100.0)
    host = CL.ClosedLoopFleet(plants, ctl, tpl, goals, rate=100.0, device_models=False)
    assert dev.device_models and not host.device_models
    xs, _ = _points(plants[0], 5, 11)
    a, b = dev._problems(xs), host._problems(xs)
    for k in ("Ad", "Bd", "wd"):
        np.testing.assert_allclose(a[k], b[k], rtol=1e-8, atol=1e-10)


@pytest.mark.gpu
def test_single_closed_loop_device_model():
    plant = D.Pendulum(D.PendulumParams())
    tpl = P_template(plant)
    ctl = CL.Controller("empc", p=3, empc=CL.EmpcSettings(num_sims=128, num_parents=16, generations=3, seed=5))
    res = CL.run_closed_loop(plant, ctl, tpl, np.zeros(2), np.array([0.8, 0.0]), 0.5, 100.0, device_model=True)
    assert np.all(np.isfinite(res.states))
    assert abs(res.states[-1, 0] - 0.8) < 0.2


def P_template(plant, T=30, umax=25.0):
    import paper_2001_04931_b200 as P

    nj = plant.m
    clin = D.linearize(plant.ode, np.zeros(plant.n), np.zeros(nj))
    return P.MpcSpec(D.discretize(clin, 0.01), T, Q=np.diag([10.0] * nj + [0.1] * nj), R=0.01 * np.eye(nj),
                     x_goal=np.zeros(plant.n), u_goal=np.zeros(nj), u_min=-umax * np.ones(nj),
                     u_max=umax * np.ones(nj))
