"""Experiment harness rows for the EMPC path on B200.

Mirrors the parts of the reference harness (``knotmpc.bench``, K/bench.py)
that touch EMPC, so its presets report B200 numbers in the reference's own
CSV schema:

* the ``empc:P:G`` controller token (K/bench.py:184-212);
* the ``key = value`` config format with list / range shorthand
  (K/bench.py:218-330);
* the trial recipe: per-(links, trial) RNG, derived seeds, start / goal
  sampling, plant and template construction (K/bench.py:336-424);
* ``solve_time_scaling`` (K/bench.py:575-615) and ``closedloop_comparison``
  (K/bench.py:618-650) rows for EMPC controllers, with the reference's
  column order and cell formatting (K/bench.py:57-94, 720-745);
* the ``closedloop_arms`` preset's EMPC arms and a solve-time preset
  (K/bench.py:855-869).

QP controller tokens (large / small / *_param) parse, but running them is
the reference's job: they are refused with ``ConfigError``.  Extensions:
``scorer`` / ``precision`` (EmpcSettings), ``device_model`` (relinearize on
the GPU) and ``draws_factory`` (inject random tensors: with FP64 and the
reference's draws the parity tests reproduce the reference's rows).

    python -m paper_2001_04931_b200.harness --preset closedloop_arms_empc --trials 1 --out rows.csv
"""

from __future__ import annotations

import argparse
import csv
import io
import os
import time
from dataclasses import dataclass, fields, replace

import numpy as np

from .closedloop import Controller, compute_metrics, cost_ratio, run_closed_loop
from .dynamics import NLinkArm, NLinkParams, Pendulum, PendulumParams, discretize, linearize
from .empc import EmpcSettings, solve_empc
from .param import KnotSchedule
from .spec import MpcSpec

EXPERIMENTS = ("param_sweep", "horizon_sweep", "robustness", "solve_time_scaling", "closedloop_comparison")
SUPPORTED = ("solve_time_scaling", "closedloop_comparison")
ROBOTS = ("pendulum", "pendulum_nograv", "nlink")

# K/bench.py:57-84 (order is the file format)
COLUMNS = [
    "experiment", "robot", "links", "T", "p", "controller", "generations", "trial", "seed", "multiplier", "start",
    "goal", "actual_cost", "cost_ratio", "normalized_cost", "rise_time", "overshoot", "itae", "opt_time_med",
    "opt_time_q1", "opt_time_q3", "mpc_time_med", "mpc_time_q1", "mpc_time_q3", "failures", "steps",
]
TIMING_COLUMNS = {"opt_time_med", "opt_time_q1", "opt_time_q3", "mpc_time_med", "mpc_time_q1", "mpc_time_q3"}


class ConfigError(ValueError):
    """A config file or mapping failed validation (K/bench.py:96-97)."""


@dataclass(frozen=True)
class ExperimentConfig:
    """The reference's experiment config (K/bench.py:100-163), EMPC fields."""

    experiment: str
    robot: str = "pendulum"
    links: tuple[int, ...] = (3,)
    T: int = 50
    controllers: tuple[str, ...] = ()
    trials: int = 20
    seed: int = 0
    duration: float = 1.0
    rate: float = 100.0
    out: str = "results.csv"
    u_max: float | None = None
    q_pos: float = 10.0
    q_vel: float = 0.1
    r_input: float = 0.01
    empc_sims: int = 1024
    empc_parents: int = 64
    # extensions
    scorer: str = "rollout"
    precision: str = "fp32"
    device_model: bool = False

    def validate(self) -> None:
        if self.experiment not in EXPERIMENTS:
            raise ConfigError(f"experiment: must be one of {', '.join(EXPERIMENTS)}; got {self.experiment!r}")
        if self.robot not in ROBOTS:
            raise ConfigError(f"robot: must be one of {', '.join(ROBOTS)}; got {self.robot!r}")
        if not self.links or any(v < 1 for v in self.links):
            raise ConfigError("links: need at least one positive link count")
        if self.T < 1:
            raise ConfigError(f"T: horizon must be >= 1, got {self.T}")
        if self.trials < 1:
            raise ConfigError(f"trials: must be >= 1, got {self.trials}")
        if self.duration <= 0:
            raise ConfigError(f"duration: must be positive, got {self.duration}")
        if self.rate <= 0:
            raise ConfigError(f"rate: must be positive, got {self.rate}")
        if self.u_max is not None and self.u_max <= 0:
            raise ConfigError(f"u_max: must be positive, got {self.u_max}")
        for tok in self.controllers:
            parse_controller_token(tok)
        for name in ("q_pos", "q_vel", "r_input"):
            if getattr(self, name) <= 0:
                raise ConfigError(f"{name}: must be positive")
        if self.empc_sims < 1 or not 1 <= self.empc_parents <= self.empc_sims:
            raise ConfigError("empc_parents: need 1 <= empc_parents <= empc_sims")
        if self.scorer not in ("rollout", "condensed") or self.precision not in ("fp32", "fp64"):
            raise ConfigError("scorer must be rollout|condensed and precision fp32|fp64")

    def resolved_controllers(self) -> tuple[str, ...]:
        if self.controllers:
            return self.controllers
        return _DEFAULT_CONTROLLERS[self.experiment]


_DEFAULT_CONTROLLERS = {
    "param_sweep": ("small", "small_param"),
    "horizon_sweep": ("small",),
    "robustness": ("small", "small_param:2", "small_param:4", "small_param:8"),
    "solve_time_scaling": ("large", "small", "large_param:5", "small_param:5"),
    "closedloop_comparison": ("large", "small_param:3", "empc:3:1", "empc:3:3"),
}


@dataclass(frozen=True)
class ControllerToken:
    kind: str
    p: int | None = None
    generations: int = 1
    text: str = ""


def _int(text: str, field_name: str) -> int:
    try:
        return int(text)
    except ValueError as e:
        raise ConfigError(f"{field_name}: expected an integer, got {text!r}") from e


def parse_controller_token(token: str) -> ControllerToken:
    """``large`` | ``small`` | ``large_param:P`` | ``small_param:P`` |
    ``empc:P:G`` (K/bench.py:184-212)."""
    kind, *args = token.split(":")
    if kind in ("large", "small"):
        if args:
            raise ConfigError(f"controllers: {token!r} takes no arguments")
        return ControllerToken(kind, text=token)
    if kind in ("large_param", "small_param"):
        if len(args) != 1:
            raise ConfigError(f"controllers: {token!r} must look like {kind}:P")
        p = _int(args[0], "controllers")
        if p < 1:
            raise ConfigError(f"controllers: knot count must be positive in {token!r}")
        return ControllerToken(kind, p=p, text=token)
    if kind == "empc":
        if len(args) != 2:
            raise ConfigError(f"controllers: {token!r} must look like empc:P:G")
        p, g = _int(args[0], "controllers"), _int(args[1], "controllers")
        if p < 1 or g < 1:
            raise ConfigError(f"controllers: knots and generations must be positive in {token!r}")
        return ControllerToken(kind, p=p, generations=g, text=token)
    raise ConfigError(f"controllers: unknown controller kind {kind!r} in {token!r}")


# ---------------------------------------------------------------------------
# key = value config files (K/bench.py:218-330)

_LISTS = {"links": int}
_SCALARS = {"experiment": str, "robot": str, "T": int, "trials": int, "seed": int, "duration": float, "rate": float,
            "out": str, "u_max": float, "q_pos": float, "q_vel": float, "r_input": float, "empc_sims": int,
            "empc_parents": int, "scorer": str, "precision": str}
# keys of the reference config that only concern its QP solvers / other experiments
_IGNORED = {"p", "horizons", "multipliers", "workers", "qp_rho", "qp_eps_prim", "qp_eps_dual", "qp_max_iters"}


def parse_list(text: str, cast, field_name: str) -> tuple:
    """Comma list with ``a:b`` (inclusive integer range) and ``a:b:step``."""
    out = []
    for chunk in (c.strip() for c in text.split(",")):
        if not chunk:
            continue
        if ":" not in chunk:
            try:
                out.append(cast(chunk))
            except ValueError as e:
                raise ConfigError(f"{field_name}: expected {cast.__name__}, got {chunk!r}") from e
            continue
        parts = chunk.split(":")
        if len(parts) not in (2, 3):
            raise ConfigError(f"{field_name}: bad range {chunk!r}, expected a:b or a:b:step")
        try:
            if cast is int and len(parts) == 2:
                out.extend(range(int(parts[0]), int(parts[1]) + 1))
                continue
            lo, hi = float(parts[0]), float(parts[1])
            step = float(parts[2]) if len(parts) == 3 else 1.0
        except ValueError as e:
            raise ConfigError(f"{field_name}: bad range {chunk!r}") from e
        if step <= 0:
            raise ConfigError(f"{field_name}: range step must be positive in {chunk!r}")
        out.extend(cast(round(lo + i * step, 12)) for i in range(int(round((hi - lo) / step)) + 1))
    if not out:
        raise ConfigError(f"{field_name}: empty list")
    return tuple(out)


def config_from_mapping(raw: dict) -> ExperimentConfig:
    if "experiment" not in raw:
        raise ConfigError("experiment: missing (this key is required)")
    kw = {}
    for key, text in raw.items():
        if key == "controllers":
            kw[key] = tuple(t.strip() for t in text.split(",") if t.strip())
        elif key == "device_model":
            kw[key] = text.strip().lower() in ("1", "true", "yes")
        elif key in _LISTS:
            kw[key] = parse_list(text, _LISTS[key], key)
        elif key in _SCALARS:
            cast = _SCALARS[key]
            try:
                kw[key] = text.strip() if cast is str else (_int(text, key) if cast is int else float(text))
            except ValueError as e:
                raise ConfigError(f"{key}: expected a number, got {text!r}") from e
        elif key not in _IGNORED:
            raise ConfigError(f"{key}: unknown config key")
    cfg = ExperimentConfig(**kw)
    cfg.validate()
    return cfg


def load_config(path: str) -> ExperimentConfig:
    """``key = value`` lines, ``#`` comments (K/bench.py:310-322)."""
    raw = {}
    with open(path, encoding="utf-8") as fh:
        for lineno, line in enumerate(fh, 1):
            line = line.split("#", 1)[0].strip()
            if not line:
                continue
            if "=" not in line:
                raise ConfigError(f"line {lineno}: expected 'key = value', got {line!r}")
            key, _, value = line.partition("=")
            raw[key.strip()] = value.strip()
    return config_from_mapping(raw)


def dump_config(cfg: ExperimentConfig) -> str:
    lines = []
    for f in fields(cfg):
        val = getattr(cfg, f.name)
        if val is None or (isinstance(val, tuple) and not val):
            continue
        lines.append(f"{f.name} = {','.join(map(str, val)) if isinstance(val, tuple) else val}")
    return "\n".join(lines) + "\n"


# ---------------------------------------------------------------------------
# trial recipe (K/bench.py:336-424): the same plants, templates and draws, so
# start / goal / seed columns equal the reference's for a given config


def make_plant(robot: str, links: int):
    if robot == "pendulum":
        return Pendulum(PendulumParams())
    if robot == "pendulum_nograv":
        return Pendulum(PendulumParams(gravity=0.0))
    if robot == "nlink":
        return NLinkArm(NLinkParams(links=links))
    raise ConfigError(f"robot: unknown robot {robot!r}")


def default_torque_bound(robot: str) -> float:
    return 25.0 if robot.startswith("pendulum") else 2.0


def make_template(plant, cfg: ExperimentConfig, T: int) -> MpcSpec:
    nj = plant.m
    bound = cfg.u_max if cfg.u_max is not None else default_torque_bound(cfg.robot)
    model = discretize(linearize(plant.ode, np.zeros(plant.n), np.zeros(nj)), 1.0 / cfg.rate)
    return MpcSpec(model=model, T=T, Q=np.diag([cfg.q_pos] * nj + [cfg.q_vel] * nj), R=cfg.r_input * np.eye(nj),
                   x_goal=np.zeros(plant.n), u_goal=np.zeros(nj), u_min=np.full(nj, -bound), u_max=np.full(nj, bound))


def trial_rng(cfg: ExperimentConfig, links: int, trial: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence(entropy=cfg.seed, spawn_key=(links, trial)))


def derived_seed(cfg: ExperimentConfig, *key: int) -> int:
    return int(np.random.SeedSequence(entropy=cfg.seed, spawn_key=tuple(key)).generate_state(1)[0])


def sample_endpoints(rng: np.random.Generator, nj: int):
    """Start and goal joint angles uniform in [-pi, pi], at rest."""
    q0 = rng.uniform(-np.pi, np.pi, nj)
    qg = rng.uniform(-np.pi, np.pi, nj)
    z = np.zeros(nj)
    return np.concatenate([q0, z]), np.concatenate([qg, z])


def _settings(cfg: ExperimentConfig, tok: ControllerToken, seed: int) -> EmpcSettings:
    return EmpcSettings(num_sims=cfg.empc_sims, num_parents=cfg.empc_parents, generations=tok.generations, seed=seed,
                        precision=cfg.precision, scorer=cfg.scorer)


def _links_of(cfg, links):
    return links if cfg.robot == "nlink" else 1


def _new_row(cfg: ExperimentConfig, links: int, trial: int) -> dict:
    row = {c: "" for c in COLUMNS}
    row.update(experiment=cfg.experiment, robot=cfg.robot, trial=trial, seed=cfg.seed, links=_links_of(cfg, links))
    return row


def _fmt_vec(v) -> str:
    return ";".join(repr(float(x)) for x in v)


def _empc_tokens(cfg):
    toks = [parse_controller_token(t) for t in cfg.resolved_controllers()]
    bad = [t.text for t in toks if t.kind != "empc"]
    if bad:
        raise ConfigError(f"controllers: {', '.join(bad)} are QP controllers; this harness runs the EMPC path "
                          "(run them with knotmpc.bench)")
    return toks


def run_solve_time_scaling(cfg: ExperimentConfig, links: int, trial: int, *, draws_factory=None) -> list[dict]:
    """Cold ``solve_empc`` wall time per EMPC token at the trial's start state
    (K/bench.py:575-615).  ``draws_factory(settings, p, m, u_min, u_max)`` ->
    ``fn(generation0, evolves, cold)`` replays injected random tensors (the
    parity seam of ``run_closed_loop``)."""
    plant = make_plant(cfg.robot, links)
    template = make_template(plant, cfg, cfg.T)
    x0, xg = sample_endpoints(trial_rng(cfg, links, trial), plant.m)
    spec = replace(template, model=discretize(linearize(plant.ode, x0, np.zeros(plant.m)), 1.0 / cfg.rate), x_goal=xg)
    rows = []
    for c_idx, tok in enumerate(_empc_tokens(cfg)):
        row = _new_row(cfg, links, trial)
        row.update(T=cfg.T, p=tok.p, controller="empc", generations=tok.generations, start=_fmt_vec(x0),
                   goal=_fmt_vec(xg), steps=1)
        st = _settings(cfg, tok, derived_seed(cfg, links, trial, c_idx))
        sched = KnotSchedule(cfg.T, tok.p)
        kw = {}
        if draws_factory is not None:
            fn = draws_factory(st, tok.p, plant.m, spec.u_min, spec.u_max)
            init, dr = fn(1, st.generations - 1, True)
            kw = dict(draws=dr, init_candidates=init)
        solve_empc(spec, sched, st, x0, **kw)  # warm the device context (graph capture, first launch)
        t0 = time.perf_counter()
        solve_empc(spec, sched, st, x0, **kw)
        elapsed = time.perf_counter() - t0
        row.update(opt_time_med=elapsed, mpc_time_med=elapsed, failures=0)
        rows.append(row)
    return rows


def run_closedloop_comparison(cfg: ExperimentConfig, links: int, trial: int, *, draws_factory=None) -> list[dict]:
    """Closed-loop runs of every EMPC token from the trial's start to its goal
    (K/bench.py:618-650); cost_ratio is relative to the first token."""
    plant = make_plant(cfg.robot, links)
    template = make_template(plant, cfg, cfg.T)
    x0, xg = sample_endpoints(trial_rng(cfg, links, trial), plant.m)
    steps = int(round(cfg.duration * cfg.rate))
    rows, base = [], None
    for c_idx, tok in enumerate(_empc_tokens(cfg)):
        st = _settings(cfg, tok, derived_seed(cfg, links, trial, c_idx))
        draws = (draws_factory(st, tok.p, plant.m, template.u_min, template.u_max)
                 if draws_factory is not None else None)
        res = run_closed_loop(plant, Controller("empc", p=tok.p, empc=st), template, x0, xg, cfg.duration, cfg.rate,
                              device_model=cfg.device_model, _draws=draws)
        rep = compute_metrics(res, template.Q, template.R, xg, cfg.rate, plant.m)
        base = rep.actual_cost if base is None else base
        row = _new_row(cfg, links, trial)
        row.update(T=cfg.T, p=tok.p, controller="empc", generations=tok.generations, start=_fmt_vec(x0),
                   goal=_fmt_vec(xg), steps=steps, actual_cost=rep.actual_cost, rise_time=rep.rise_time,
                   overshoot=rep.overshoot, itae=rep.itae, opt_time_q1=rep.opt_time_quartiles[0],
                   opt_time_med=rep.opt_time_quartiles[1], opt_time_q3=rep.opt_time_quartiles[2],
                   mpc_time_q1=rep.mpc_time_quartiles[0], mpc_time_med=rep.mpc_time_quartiles[1],
                   mpc_time_q3=rep.mpc_time_quartiles[2], failures=rep.failures,
                   cost_ratio=cost_ratio(rep.actual_cost, base))
        rows.append(row)
    return rows


_RUNNERS = {"solve_time_scaling": run_solve_time_scaling, "closedloop_comparison": run_closedloop_comparison}


def _row_key(row):
    return (str(row["experiment"]), row["links"] if row["links"] != "" else 0, str(row["controller"]), str(row["p"]),
            str(row["generations"]), str(row["T"]), str(row["multiplier"]), row["trial"])


def run_experiment(cfg: ExperimentConfig, out_dir: str | None = ".", *, draws_factory=None) -> list[dict]:
    """Every (links, trial) of an EMPC experiment, rows sorted like the
    reference's (K/bench.py:770-790); writes ``cfg.out`` unless out_dir is None.
    One process drives the GPU (the reference's process pool parallelises CPU
    trials; here the device is the parallel resource)."""
    cfg.validate()
    if cfg.experiment not in SUPPORTED:
        raise ConfigError(f"experiment: {cfg.experiment!r} has no EMPC rows; supported: {', '.join(SUPPORTED)}")
    run = _RUNNERS[cfg.experiment]
    links_axis = cfg.links if cfg.robot == "nlink" else (1,)
    rows = [r for links in links_axis for trial in range(cfg.trials)
            for r in run(cfg, links, trial, draws_factory=draws_factory)]
    rows.sort(key=_row_key)
    if out_dir is not None:
        os.makedirs(out_dir, exist_ok=True)
        write_csv(os.path.join(out_dir, cfg.out), rows)
    return rows


def _fmt_cell(val) -> str:
    return repr(val) if isinstance(val, float) else str(val)


def write_csv(path: str, rows: list[dict]) -> None:
    """RFC-4180, UTF-8, the reference's fixed column order (K/bench.py:720-733)."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(COLUMNS)
        for row in rows:
            w.writerow([_fmt_cell(row[c]) for c in COLUMNS])


def rows_to_csv_text(rows: list[dict], include_timing: bool = True) -> str:
    buf = io.StringIO()
    cols = [c for c in COLUMNS if include_timing or c not in TIMING_COLUMNS]
    w = csv.writer(buf)
    w.writerow(cols)
    for row in rows:
        w.writerow([_fmt_cell(row[c]) for c in cols])
    return buf.getvalue()


# ---------------------------------------------------------------------------
# presets: the EMPC arms of the reference's presets (K/bench.py:839-869)

PRESETS = {
    "closedloop_arms_empc": (
        lambda: ExperimentConfig(experiment="closedloop_comparison", robot="nlink", links=(1, 2, 4, 6), T=100,
                                 controllers=("empc:3:1", "empc:3:3"), trials=5, duration=10.0, rate=100.0, seed=1008,
                                 out="closedloop_arms_empc.csv"),
        "EMPC arms of closedloop_arms (convex arms run in knotmpc.bench)"),
    "solve_times_empc_t50": (
        lambda: ExperimentConfig(experiment="solve_time_scaling", robot="nlink", links=tuple(range(1, 14)), T=50,
                                 controllers=("empc:5:1", "empc:5:3", "empc:5:10"), trials=20, rate=100.0, seed=1006,
                                 out="solve_times_empc_t50.csv"),
        "EMPC solve times vs links at horizon 50 (the solve_times_t50 robots and trials)"),
}


def preset_config(name: str) -> ExperimentConfig:
    if name not in PRESETS:
        raise ConfigError(f"unknown preset {name!r}; available: {', '.join(sorted(PRESETS))}")
    return PRESETS[name][0]()


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    g = ap.add_mutually_exclusive_group(required=True)
    g.add_argument("--preset", choices=sorted(PRESETS))
    g.add_argument("--config")
    ap.add_argument("--trials", type=int)
    ap.add_argument("--links", help="override, e.g. 1,2 or 1:6")
    ap.add_argument("--duration", type=float)
    ap.add_argument("--out")
    ap.add_argument("--out-dir", default=".")
    ap.add_argument("--scorer", choices=["rollout", "condensed"])
    ap.add_argument("--device-model", action="store_true")
    a = ap.parse_args(argv)
    cfg = preset_config(a.preset) if a.preset else load_config(a.config)
    over = {}
    if a.trials:
        over["trials"] = a.trials
    if a.links:
        over["links"] = parse_list(a.links, int, "links")
    if a.duration:
        over["duration"] = a.duration
    if a.out:
        over["out"] = a.out
    if a.scorer:
        over["scorer"] = a.scorer
    if a.device_model:
        over["device_model"] = True
    cfg = replace(cfg, **over)
    rows = run_experiment(cfg, a.out_dir)
    print(f"{len(rows)} rows -> {os.path.join(a.out_dir, cfg.out)}")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
