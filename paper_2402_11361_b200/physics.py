"""Gas/flow parameters, conserved-state helpers and the reference's error types.

Follows ``physics.py`` of the reference (FlowParams physics.py:32-73,
AdmissibilityError physics.py:23-29, conserved physics.py:108-119,
boundary_operator physics.py:204-223) for any dimension d in {2, 3}: the
conserved state is (rho, rho*v_1..rho*v_d, rho*E), ns = d + 2, and the bulk
viscosity ratio is lambda = -2/d.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class AdmissibilityError(RuntimeError):
    """State left the admissible set (rho > 0, pressure > 0) (physics.py:23)."""

    def __init__(self, component: str, value: float):
        self.component = component
        self.value = value
        super().__init__(f"inadmissible state: {component} = {value:.6g}")


@dataclass(frozen=True)
class FlowParams:
    """Nondimensional parameters; same fields and defaults as physics.py:32-57."""

    gamma: float = 1.4
    prandtl: float = 0.71
    reynolds_acoustic: float = 1.0
    mach_ref: float = 0.1
    mu: float = 1.0
    reynolds_flow: float | None = None

    def __post_init__(self):
        if self.gamma <= 1.0:
            raise ValueError("gamma must exceed 1")
        if self.prandtl <= 0 or self.reynolds_acoustic <= 0:
            raise ValueError("Pr and Re must be positive")
        if self.reynolds_flow is None:
            object.__setattr__(self, "reynolds_flow", self.reynolds_acoustic * self.mach_ref)

    @property
    def R(self) -> float:
        return (self.gamma - 1.0) / self.gamma

    @property
    def c_p(self) -> float:
        return 1.0

    @property
    def c_v(self) -> float:
        return self.R / (self.gamma - 1.0)


def lambda_bulk(dim: int) -> float:
    return -2.0 / dim


def conserved(rho, v, P, params: FlowParams) -> np.ndarray:
    """Conserved state from (rho, velocity (..., d), pressure)."""
    rho = np.asarray(rho, dtype=float)
    v = np.asarray(v, dtype=float)
    P = np.asarray(P, dtype=float)
    d = v.shape[-1]
    u = np.empty(np.broadcast_shapes(rho.shape, v.shape[:-1], P.shape) + (d + 2,))
    u[..., 0] = rho
    u[..., 1 : d + 1] = rho[..., None] * v
    u[..., d + 1] = P / (params.gamma - 1.0) + 0.5 * rho * np.einsum("...i,...i->...", v, v)
    return u


def check_admissible_host(u: np.ndarray, gamma: float) -> None:
    """Host-side admissibility check (physics.py:85-94), any dimension."""
    u = np.atleast_2d(u)
    d = u.shape[-1] - 2
    rho = u[..., 0]
    if np.any(rho <= 0.0) or not np.all(np.isfinite(rho)):
        raise AdmissibilityError("rho", float(np.min(rho)))
    kin = 0.5 * np.einsum("...i,...i->...", u[..., 1 : d + 1], u[..., 1 : d + 1]) / rho
    pres = (gamma - 1.0) * (u[..., d + 1] - kin)
    if np.any(pres <= 0.0) or not np.all(np.isfinite(pres)):
        raise AdmissibilityError("pressure", float(np.min(pres)))


# boundary kinds: the reference's two plus the moving isothermal wall that the
# 2D Couette config needs (a wall with velocity u_w; u_w = 0 is the
# reference's isothermal_noslip_wall, physics.py:214-222)
BOUNDARY_KINDS = ("dirichlet_state", "isothermal_noslip_wall", "isothermal_moving_wall")
