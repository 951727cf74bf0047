"""Host-side model types, plants and the synthetic-system generator.

Mirrors the parts of knotmpc.dynamics (K/dynamics.py) the EMPC path and its
closed loop consume: ``DiscreteLinearModel`` (K/dynamics.py:223-238), the
plants (``Pendulum`` K/dynamics.py:33-75, ``NLinkArm`` K/dynamics.py:90-199),
``linearize`` (K/dynamics.py:241-262), ``discretize`` (K/dynamics.py:265-290)
and the RK4 ground-truth integrator (K/dynamics.py:316-330).  Model generation is host FP64 work
outside the timed solve, exactly as in the paper and the
reference harness (K/closedloop.py:76-79).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ContinuousLinearModel:
    """xdot = A x + B u + w."""

    A: np.ndarray
    B: np.ndarray
    w: np.ndarray

    @property
    def n(self) -> int:
        return self.A.shape[0]

    @property
    def m(self) -> int:
        return self.B.shape[1]


@dataclass(frozen=True)
class DiscreteLinearModel:
    """x[k+1] = Ad x[k] + Bd u[k] + wd (K/dynamics.py:223-238)."""

    Ad: np.ndarray
    Bd: np.ndarray
    wd: np.ndarray
    dt: float

    @property
    def n(self) -> int:
        return self.Ad.shape[0]

    @property
    def m(self) -> int:
        return self.Bd.shape[1]


@dataclass(frozen=True)
class NLinkParams:
    """Planar serial chain with point masses at the link tips (K/dynamics.py:90-112)."""

    links: int
    mass: float | np.ndarray = 1.0
    length: float | np.ndarray = 0.25
    damping: float = 0.01
    gravity: float = 0.0

    def __post_init__(self):
        if self.links < 1:
            raise ValueError("links must be >= 1")
        for name in ("mass", "length"):
            v = np.broadcast_to(np.asarray(getattr(self, name), float), (self.links,)).copy()
            if np.any(v <= 0):
                raise ValueError("masses and lengths must be positive")
            object.__setattr__(self, name, v)
        if self.damping < 0:
            raise ValueError("damping must be non-negative")


class NLinkArm:
    """State x = [q, qdot], one torque per joint.

    Lagrangian in absolute link angles th = cumsum(q): with G[j,k] the mass
    carried at or beyond link max(j,k), the inertia in th-coordinates is
    G l_j l_k cos(th_j - th_k); the velocity terms are G l_j l_k
    sin(th_j - th_k) thd_k^2 and gravity g l_j cos(th_j) sum_{i>=j} m_i.  Joint
    torques and damping map to th-coordinates through the transpose of the
    cumulative-sum map, and joint accelerations are its inverse (differences).
    """

    def __init__(self, params: NLinkParams):
        self.params = params
        self.n = 2 * params.links
        self.m = params.links
        mass = params.mass
        self._carried = np.cumsum(mass[::-1])[::-1]  # sum_{i >= j} m_i
        j = np.arange(params.links)
        self._G = self._carried[np.maximum.outer(j, j)]
        self._ll = np.outer(params.length, params.length)

    def accel(self, q, qd, tau):
        p = self.params
        th = np.cumsum(q)
        thd = np.cumsum(qd)
        dth = th[:, None] - th[None, :]
        GL = self._G * self._ll
        M = GL * np.cos(dth)
        coriolis = (GL * np.sin(dth)) @ (thd * thd)
        grav = p.gravity * self._carried * p.length * np.cos(th)
        f = tau - p.damping * qd
        y = f.copy()
        y[:-1] -= f[1:]  # generalized force in absolute coordinates
        thdd = np.linalg.solve(M, y - coriolis - grav)
        qdd = thdd.copy()
        qdd[1:] -= thdd[:-1]
        return qdd

    def ode(self, x, u):
        L = self.params.links
        x = np.asarray(x, float)
        return np.concatenate([x[L:], self.accel(x[:L], x[L:], np.asarray(u, float))])


def linearize(f, x0, u0, eps: float = 1e-6) -> ContinuousLinearModel:
    """Central-difference Jacobians with the affine residual (K/dynamics.py:241-262)."""
    x0 = np.asarray(x0, float)
    u0 = np.asarray(u0, float)
    n, m = x0.size, u0.size
    A = np.empty((n, n))
    B = np.empty((n, m))
    for i in range(n):
        dx = np.zeros(n)
        dx[i] = eps
        A[:, i] = (f(x0 + dx, u0) - f(x0 - dx, u0)) / (2 * eps)
    for j in range(m):
        du = np.zeros(m)
        du[j] = eps
        B[:, j] = (f(x0, u0 + du) - f(x0, u0 - du)) / (2 * eps)
    w = np.asarray(f(x0, u0), float) - A @ x0 - B @ u0
    return ContinuousLinearModel(A, B, w)


def discretize(model: ContinuousLinearModel, dt: float, method: str = "exact") -> DiscreteLinearModel:
    """Zero-order-hold discretization via the augmented matrix exponential
    (K/dynamics.py:265-290); ``euler`` gives I + A dt."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    n, m = model.n, model.m
    if method == "euler":
        return DiscreteLinearModel(np.eye(n) + model.A * dt, model.B * dt, model.w * dt, dt)
    if method != "exact":
        raise ValueError(f"unknown discretization method {method!r}")
    from scipy.linalg import expm

    aug = np.zeros((n + m + 1, n + m + 1))
    aug[:n, :n] = model.A
    aug[:n, n:n + m] = model.B
    aug[:n, -1] = model.w
    E = expm(aug * dt)
    return DiscreteLinearModel(E[:n, :n], E[:n, n:n + m], E[:n, -1], dt)


@dataclass(frozen=True)
class PendulumParams:
    """m l^2 qdd + b qd + m g l sin(q) = tau, q from the hanging position
    (K/dynamics.py:33-48)."""

    mass: float = 1.0
    length: float = 1.0
    damping: float = 0.05
    gravity: float = 9.81

    def __post_init__(self):
        if self.mass <= 0 or self.length <= 0:
            raise ValueError("mass and length must be positive")
        if self.damping < 0:
            raise ValueError("damping must be non-negative")


class Pendulum:
    """Single-joint plant, state [q, qd], one torque input (K/dynamics.py:59-75)."""

    n = 2
    m = 1

    def __init__(self, params: PendulumParams = PendulumParams()):
        self.params = params

    def ode(self, x, u):
        p = self.params
        q, qd = float(x[0]), float(x[1])
        inertia = p.mass * p.length**2
        qdd = (float(u[0]) - p.damping * qd - p.mass * p.gravity * p.length * np.sin(q)) / inertia
        return np.array([qd, qdd])


def rk4_step(f, x, u, dt: float) -> np.ndarray:
    """Classic RK4 with the input held over the step (K/dynamics.py:316-322)."""
    h2 = 0.5 * dt
    k1 = f(x, u)
    k2 = f(x + h2 * k1, u)
    k3 = f(x + h2 * k2, u)
    k4 = f(x + dt * k3, u)
    return x + (dt / 6.0) * (k1 + 2 * k2 + 2 * k3 + k4)


def integrate(f, x, u, dt: float, substeps: int = 10) -> np.ndarray:
    """One zero-order-hold control period as ``substeps`` RK4 steps
    (K/dynamics.py:325-330)."""
    h = dt / substeps
    for _ in range(substeps):
        x = rk4_step(f, x, u, h)
    return x


def linearize_discretize(plant, xs, us=None, dt: float = 0.01, method: str = "exact", eps: float = 1e-6,
                         device: int = 0):
    """Batched ``discretize(linearize(plant.ode, x, u, eps), dt, method)`` on
    the GPU (K/dynamics.py:241-290): one CTA per operating point
    computes the central-difference Jacobians of the plant ODE and the
    zero-order-hold exponential of the augmented matrix in FP64.

    ``plant`` is a ``Pendulum`` or an ``NLinkArm`` (the reference's plant
    models; an arbitrary Python callable cannot run on the device -- use
    ``linearize`` / ``discretize`` for those).  ``xs`` is (I, n), ``us`` (I, m)
    (default zeros, the closed loop's nominal input).  Returns stacked
    ``(Ad (I,n,n), Bd (I,n,m), wd (I,n))``.
    """
    from . import _native as nat

    if method not in ("exact", "euler"):
        raise ValueError(f"unknown discretization method {method!r}")
    if dt <= 0:
        raise ValueError("dt must be positive")
    dev_plant = _device_plant(plant)
    xs = np.atleast_2d(np.asarray(xs, float))
    us = np.zeros((xs.shape[0], plant.m)) if us is None else np.atleast_2d(np.asarray(us, float))
    if xs.shape[1] != plant.n or us.shape != (xs.shape[0], plant.m):
        raise ValueError("xs must be (I, n) and us (I, m)")
    meth = nat.EMPC_DISCRETIZE_EXACT if method == "exact" else nat.EMPC_DISCRETIZE_EULER
    return nat.plant_linearize_discretize(*dev_plant, xs, us, eps, dt, meth, device)


def _device_plant(plant):
    """(kind, links, mass, length, damping, gravity) of a plant the device knows."""
    from . import _native as nat

    if isinstance(plant, Pendulum):
        p = plant.params
        return nat.EMPC_PLANT_PENDULUM, 1, [p.mass], [p.length], p.damping, p.gravity
    if isinstance(plant, NLinkArm):
        p = plant.params
        return nat.EMPC_PLANT_NLINK, p.links, p.mass, p.length, p.damping, p.gravity
    raise TypeError(f"no device model for plant type {type(plant).__name__}")


def integrate_batch(plant, xs, us, dt: float, substeps: int = 10, device: int = 0) -> np.ndarray:
    """``integrate(plant.ode, x, u, dt, substeps)`` for every row of ``xs`` /
    ``us`` on the GPU, one warp per instance (K/dynamics.py:316-330)."""
    from . import _native as nat

    xs = np.atleast_2d(np.asarray(xs, float))
    us = np.atleast_2d(np.asarray(us, float))
    if xs.shape[1] != plant.n or us.shape != (xs.shape[0], plant.m):
        raise ValueError("xs must be (I, n) and us (I, m)")
    return nat.plant_integrate(*_device_plant(plant), xs, us, dt, substeps, device)
