"""Closed-loop EMPC on the B200 path.

Drop-in for the EMPC branch of ``knotmpc.closedloop.run_closed_loop``
(K/closedloop.py:59-133): every control period the controller's plant model
is relinearized at the measured state with zero nominal input
(K/closedloop.py:103), discretized exactly at the control rate
(K/closedloop.py:104), and handed to ``solve_empc`` warm-started from the
previous period's population (K/closedloop.py:109-111).  The clipped first
knot is held for one period while the true plant is integrated with RK4
substeps (K/closedloop.py:113, 128-130).

B200 specifics: the population never leaves the GPU between periods -- each
warm solve re-scores the device-resident population of the previous period
at the new state (one cooperative launch for single problems), so a period
uploads only the relinearized (A_d, B_d, w_d), x0 and sigma and reads back
u and the best knots.  ``ClosedLoopFleet`` steps many independent plants
(C5-style) with one batched solve per period.

The QP controllers of the reference (kinds large/small/large_param/
small_param, K/closedloop.py:114-126) are outside the EMPC hot path and are
not provided; asking for one raises ``NotImplementedError``.

The response metrics (K/closedloop.py:160-300) are plain host numpy and are
restated here so a user of the reference's closed-loop study finds them
next to the runner.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, replace

import numpy as np

from .dynamics import DiscreteLinearModel, NLinkArm, NLinkParams, Pendulum, PendulumParams, discretize, integrate, \
    integrate_batch, linearize, linearize_discretize
from .empc import EmpcBatch, EmpcSettings, solve_empc
from .param import KnotSchedule

_KINDS = ("large", "small", "large_param", "small_param", "empc")


@dataclass(frozen=True)
class Controller:
    """Solver inside the loop (K/closedloop.py:30-49); only ``empc`` runs here."""

    kind: str
    p: int | None = None
    empc: EmpcSettings | None = None

    def __post_init__(self):
        if self.kind not in _KINDS:
            raise ValueError(f"unknown controller kind {self.kind!r}")
        if self.kind in ("large_param", "small_param", "empc") and self.p is None:
            raise ValueError(f"{self.kind} needs a knot count p")
        if self.kind == "empc" and self.empc is None:
            object.__setattr__(self, "empc", EmpcSettings())


@dataclass
class SimResult:
    """(K/closedloop.py:52-58)"""

    states: np.ndarray  # (H+1, n)
    inputs: np.ndarray  # (H, m)
    opt_time: np.ndarray  # per-period solve time, s
    mpc_time: np.ndarray  # same as opt_time for EMPC (no matrix construction)
    failures: int  # always 0: EMPC returns a solution every period


def run_closed_loop(plant, controller: Controller, template, x0, x_goal, duration: float, rate: float, *,
                    controller_plant=None, qp_settings=None, plant_substeps: int = 10,
                    device_model: bool = False, _draws=None) -> SimResult:
    """Simulate ``duration`` s of EMPC at ``rate`` Hz (K/closedloop.py:59-133).

    ``controller_plant`` (default: the true plant) is only ever linearized.
    Linearization and discretization are excluded from the timing columns
    (K/closedloop.py:76-79).  ``_draws(generation0, evolves, init)`` -> (init
    candidates or None, list of per-evolve draws) is the parity seam that
    replays the reference's random tensors.  ``device_model=True`` (an
    extension) relinearizes and discretizes a ``Pendulum`` / ``NLinkArm``
    controller model on the GPU (``dynamics.linearize_discretize``, SURVEY §8
    f3) instead of the host ``linearize`` + ``expm``.
    """
    if controller.kind != "empc":
        raise NotImplementedError(f"controller kind {controller.kind!r} is a QP solver outside the B200 EMPC path")
    H = int(round(duration * rate))
    dt = 1.0 / rate
    model_src = controller_plant if controller_plant is not None else plant
    x_goal = np.asarray(x_goal, float)
    n, m = plant.n, plant.m
    states = np.empty((H + 1, n))
    inputs = np.empty((H, m))
    opt_time = np.zeros(H)
    states[0] = np.asarray(x0, float)
    sched = KnotSchedule(template.T, controller.p)
    st = controller.empc
    u_nom = np.zeros(m)
    population = None
    x = states[0].copy()
    for i in range(H):
        if device_model:
            Ad, Bd, wd = linearize_discretize(model_src, x[None], None, dt, "exact")
            model = DiscreteLinearModel(Ad[0], Bd[0], wd[0], dt)
        else:
            model = discretize(linearize(model_src.ode, x, u_nom), dt, "exact")
        spec = replace(template, model=model, x_goal=x_goal)
        kw = {}
        if _draws is not None:
            cold = population is None
            g0 = 1 if cold else population.generation
            init_c, dr = _draws(g0, st.generations - 1 if cold else st.generations, cold)
            kw = dict(draws=dr, init_candidates=init_c)
        t0 = time.perf_counter()
        res = solve_empc(spec, sched, st, x, prev=population, **kw)
        opt_time[i] = time.perf_counter() - t0
        population = res.population
        u = np.clip(res.u, spec.u_min, spec.u_max)
        inputs[i] = u
        x = integrate(plant.ode, x, u, dt, substeps=plant_substeps)
        states[i + 1] = x
    return SimResult(states, inputs, opt_time, opt_time.copy(), 0)


class ClosedLoopFleet:
    """Many independent plants of one shape under EMPC, one batched device
    solve per control period (the C5 fleet: K/bench.py:688-705 runs these as
    a process pool of ``run_closed_loop`` calls).

    ``plants`` and ``x_goals`` are per instance; all share ``template``'s
    T/Q/R/bounds and one schedule.  The populations stay on the GPU.  When
    every controller model is the same ``Pendulum`` / ``NLinkArm`` the
    relinearization + discretization of all instances runs as one batched
    device call (``dynamics.linearize_discretize``) instead of
    I host ``linearize`` + ``expm`` calls.
    """

    def __init__(self, plants, controller: Controller, template, x_goals, rate: float, *, controller_plants=None,
                 plant_substeps: int = 10, device_models: bool = True):
        if controller.kind != "empc":
            raise NotImplementedError("ClosedLoopFleet runs EMPC controllers only")
        self.plants = list(plants)
        self.models = list(controller_plants) if controller_plants is not None else self.plants
        self.I = len(self.plants)
        self.template, self.controller, self.rate = template, controller, rate
        self.sched = KnotSchedule(template.T, controller.p)
        self.x_goals = np.broadcast_to(np.asarray(x_goals, float), (self.I, self.plants[0].n)).copy()
        self.substeps = plant_substeps
        self.population = None
        self.batch = None
        def uniform(ps):
            return isinstance(ps[0], (Pendulum, NLinkArm)) and all(
                type(q) is type(ps[0]) and (q is ps[0] or _same_params(q.params, ps[0].params)) for q in ps)

        self.device_models = device_models and uniform(self.models)
        self.device_plants = device_models and uniform(self.plants)

    def _problems(self, xs):
        dt = 1.0 / self.rate
        t = self.template
        I = self.I
        if self.device_models:
            Ad, Bd, wd = linearize_discretize(self.models[0], xs, None, dt, "exact")
        else:
            mods = [discretize(linearize(mdl.ode, x, np.zeros(mdl.m)), dt, "exact") for mdl, x in zip(self.models, xs)]
            Ad, Bd, wd = (np.stack([d.Ad for d in mods]), np.stack([d.Bd for d in mods]),
                          np.stack([d.wd for d in mods]))
        bc = lambda v, shape: np.broadcast_to(np.asarray(v, float), shape)  # noqa: E731
        n, m = self.plants[0].n, self.plants[0].m
        return {"Ad": Ad, "Bd": Bd, "wd": wd, "Q": bc(t.Q, (I, n, n)), "R": bc(t.R, (I, m, m)),
                "x_goal": self.x_goals, "u_goal": bc(t.u_goal, (I, m)), "u_min": bc(t.u_min, (I, m)),
                "u_max": bc(t.u_max, (I, m))}

    def step(self, xs):
        """One control period: relinearize all plants, one batched warm solve,
        integrate every plant.  Returns (next states, inputs, solve seconds)."""
        xs = np.asarray(xs, float)
        probs = self._problems(xs)
        if self.batch is None:
            self.batch = EmpcBatch(probs, self.sched, self.controller.empc)
        else:
            self.batch.probs = {k: np.ascontiguousarray(v) for k, v in probs.items()}
        t0 = time.perf_counter()
        r = self.batch.solve(xs, prev=self.population)
        dt_solve = time.perf_counter() - t0
        self.population = r.population
        u = np.clip(r.u, probs["u_min"], probs["u_max"])
        if self.device_plants:
            nxt = integrate_batch(self.plants[0], xs, u, 1.0 / self.rate, self.substeps)
        else:
            nxt = np.stack([integrate(pl.ode, x, ui, 1.0 / self.rate, substeps=self.substeps)
                            for pl, x, ui in zip(self.plants, xs, u)])
        return nxt, u, dt_solve

    def run(self, x0s, duration: float) -> list[SimResult]:
        H = int(round(duration * self.rate))
        x = np.broadcast_to(np.asarray(x0s, float), (self.I, self.plants[0].n)).copy()
        states = np.empty((self.I, H + 1, x.shape[1]))
        inputs = np.empty((self.I, H, self.plants[0].m))
        tm = np.zeros(H)
        states[:, 0] = x
        for i in range(H):
            x, u, tm[i] = self.step(x)
            states[:, i + 1] = x
            inputs[:, i] = u
        return [SimResult(states[k], inputs[k], tm.copy(), tm.copy(), 0) for k in range(self.I)]


def _same_params(a, b) -> bool:
    for f in ("mass", "length", "damping", "gravity"):
        if not np.array_equal(np.asarray(getattr(a, f)), np.asarray(getattr(b, f))):
            return False
    return True


# ---------------------------------------------------------------------------
# robustness helper and response metrics (host numpy)


def apply_error_multiplier(params, multiplier: float):
    """Deliberately wrong controller model (K/closedloop.py:140-156): pendulum
    mass and length scale together, N-link tip masses scale."""
    if multiplier <= 0:
        raise ValueError("multiplier must be positive")
    if isinstance(params, PendulumParams):
        return replace(params, mass=params.mass * multiplier, length=params.length * multiplier)
    if isinstance(params, NLinkParams):
        return replace(params, mass=params.mass * multiplier)
    raise TypeError(f"unknown parameter type {type(params)!r}")


def actual_cost(states, inputs, Q, R, x_goal, u_goal=None) -> float:
    """Realized tracking cost, final stage padded with u = 0 (K/closedloop.py:163-173)."""
    X = np.asarray(states, float)
    U = np.asarray(inputs, float)
    ug = np.zeros(U.shape[1]) if u_goal is None else np.asarray(u_goal, float)
    U = np.concatenate([U, np.zeros((1, U.shape[1]))])
    ex = np.asarray(x_goal, float) - X
    eu = ug - U
    return float(np.einsum("ti,ij,tj->", ex, np.asarray(Q, float), ex)
                 + np.einsum("ti,ij,tj->", eu, np.asarray(R, float), eu))


def cost_ratio(cost: float, baseline: float) -> float:
    """(K/closedloop.py:176-180)"""
    return np.nan if baseline == 0.0 else cost / baseline


def normalized_cost(cost: float, cost_at_unity: float) -> float:
    """(K/closedloop.py:183-186)"""
    return cost_ratio(cost, cost_at_unity)


def _per_joint(positions, start, goal):
    return (np.atleast_2d(np.asarray(positions, float)), np.atleast_1d(np.asarray(start, float)),
            np.atleast_1d(np.asarray(goal, float)))


def rise_time(positions, start, goal, rate: float) -> np.ndarray:
    """First sample at or past 90 % of the step, per joint, in s; NaN if never
    (K/closedloop.py:189-207)."""
    pos, start, goal = _per_joint(positions, start, goal)
    out = np.full(start.size, np.nan)
    for j in range(start.size):
        d = goal[j] - start[j]
        if d == 0:
            out[j] = 0.0
            continue
        idx = np.flatnonzero((pos[:, j] - (start[j] + 0.9 * d)) * np.sign(d) >= 0)
        if idx.size:
            out[j] = idx[0] / rate
    return out


def percent_overshoot(positions, start, goal) -> np.ndarray:
    """Peak excursion past the goal as % of the step, per joint; NaN for a zero
    step (K/closedloop.py:210-225)."""
    pos, start, goal = _per_joint(positions, start, goal)
    out = np.full(start.size, np.nan)
    for j in range(start.size):
        d = goal[j] - start[j]
        if d != 0:
            out[j] = max(0.0, float(np.max((pos[:, j] - goal[j]) * np.sign(d)))) / abs(d) * 100.0
    return out


def itae(positions, command, rate: float, t_start: float = 0.0, t_end: float | None = None) -> np.ndarray:
    """Trapezoidal integral of t*|error| per joint (K/closedloop.py:228-243)."""
    pos = np.atleast_2d(np.asarray(positions, float))
    cmd = np.asarray(command, float)
    if cmd.ndim < 2:
        cmd = np.broadcast_to(np.atleast_1d(cmd), pos.shape)
    t = np.arange(pos.shape[0]) / rate
    hi = t[-1] if t_end is None else t_end
    sel = (t >= t_start) & (t <= hi)
    return np.trapezoid((t[sel] - t_start)[:, None] * np.abs(cmd[sel] - pos[sel]), t[sel], axis=0)


@dataclass
class MetricsReport:
    """(K/closedloop.py:246-255)"""

    actual_cost: float
    rise_time: float
    overshoot: float
    itae: float
    opt_time_quartiles: tuple[float, float, float]
    mpc_time_quartiles: tuple[float, float, float]
    failures: int


def compute_metrics(result: SimResult, spec_Q, spec_R, x_goal, rate: float, n_joints: int) -> MetricsReport:
    """Joint-level medians of the response metrics (K/closedloop.py:258-279)."""
    x0 = result.states[0]
    pos = result.states[:, :n_joints]
    qs = lambda a: tuple(float(v) for v in np.percentile(a, [25, 50, 75]))  # noqa: E731
    return MetricsReport(
        actual_cost=actual_cost(result.states, result.inputs, spec_Q, spec_R, x_goal),
        rise_time=float(np.median(rise_time(pos, x0[:n_joints], x_goal[:n_joints], rate))),
        overshoot=float(np.median(percent_overshoot(pos, x0[:n_joints], x_goal[:n_joints]))),
        itae=float(np.median(itae(pos, x_goal[:n_joints], rate))),
        opt_time_quartiles=qs(result.opt_time),
        mpc_time_quartiles=qs(result.mpc_time),
        failures=result.failures,
    )
