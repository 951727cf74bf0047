"""The MPC problem statement (mirror of knotmpc.condense.MpcSpec, K/condense.py:42-87).

Same fields, broadcasting and validation errors as the reference, so a spec
built for either package is accepted by the other (the solver only reads
attributes).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .dynamics import DiscreteLinearModel


@dataclass(frozen=True)
class MpcSpec:
    model: DiscreteLinearModel
    T: int
    Q: np.ndarray
    R: np.ndarray
    x_goal: np.ndarray
    u_goal: np.ndarray
    u_min: np.ndarray
    u_max: np.ndarray
    x_min: np.ndarray | None = None
    x_max: np.ndarray | None = None

    def __post_init__(self):
        n, m = self.model.n, self.model.m
        if self.T < 1:
            raise ValueError("horizon must be at least one step")
        for name, size in (("x_goal", n), ("u_goal", m), ("u_min", m), ("u_max", m)):
            object.__setattr__(self, name, np.broadcast_to(np.asarray(getattr(self, name), float), (size,)).copy())
        for name in ("Q", "R"):
            object.__setattr__(self, name, np.asarray(getattr(self, name), float))
        if self.Q.shape != (n, n) or self.R.shape != (m, m):
            raise ValueError("Q and R must match the model dimensions")
        _check_symmetric(self.Q, "Q")
        _check_symmetric(self.R, "R")
        if np.min(np.linalg.eigvalsh(self.Q)) < -1e-9:
            raise ValueError("Q must be positive semidefinite")
        if np.min(np.linalg.eigvalsh(self.R)) <= 0:
            raise ValueError("R must be positive definite")
        if np.any(self.u_min > self.u_max):
            raise ValueError("u_min must be elementwise <= u_max")
        for name in ("x_min", "x_max"):
            val = getattr(self, name)
            if val is not None:
                object.__setattr__(self, name, np.broadcast_to(np.asarray(val, float), (n,)).copy())

    @property
    def has_state_bounds(self) -> bool:
        return (self.x_min is not None and bool(np.any(np.isfinite(self.x_min)))) or (
            self.x_max is not None and bool(np.any(np.isfinite(self.x_max))))


def _check_symmetric(M, name):
    if np.max(np.abs(M - M.T)) > 1e-9 * (1.0 + np.max(np.abs(M))):
        raise ValueError(f"{name} must be symmetric")
