"""Benchmark case definitions (host setup).

3D cases restate the reference's ``cases.py`` (CouetteCase cases.py:21-107,
TgvCase cases.py:110-158).  2D cases are the BASELINE.json configs the
reference cannot run:

* ``CouettePlane2D`` -- C1: plane compressible Couette flow between an
  isothermal no-slip wall (y=0) and an isothermal wall moving at u_w (y=H),
  x-periodic.  Acoustic scaling (c_inf = 1, T_inf = 1, u_w = M), both walls at
  T_w = 1 (BASELINE leaves the wall temperatures unspecified).
* ``UniformFlow2D`` -- C2: uniform flow rho=1, v=(1, 0.3), P=1/(gamma M^2) with
  flow scaling as CouetteCase (Re_acoustic = Re_flow = Re, mach_ref = M).
* ``SphereCase`` -- C4 (3D, the reference has neither the mesh nor the wall
  BC): steady flow past a unit-diameter sphere on the O-grid of
  ``mesh.build_sphere_ogrid_mesh``; adiabatic no-slip sphere, free-stream
  Dirichlet far field.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import BOUNDARY_LABELS
from .physics import FlowParams, conserved


@dataclass
class CouetteCase:
    """Manufactured 3D Couette solution on the unit cube (cases.py:21-107)."""

    alpha_c: float = 0.8
    beta_c: float = 0.85
    gamma: float = 1.4
    prandtl: float = 0.71
    mach: float = 0.15
    reynolds: float = 1.0
    rho_inf: float = 1.0
    params: FlowParams = field(init=False)

    def __post_init__(self):
        self.params = FlowParams(gamma=self.gamma, prandtl=self.prandtl, reynolds_acoustic=self.reynolds,
                                 mach_ref=self.mach, reynolds_flow=self.reynolds)

    @property
    def t_inf(self):
        return 1.0 / ((self.gamma - 1.0) * self.mach**2)

    @property
    def p_inf(self):
        return self.rho_inf * self.t_inf / self.gamma

    def temperature(self, y):
        g = self.gamma
        return self.t_inf * (self.alpha_c + y * (self.beta_c - self.alpha_c)
                             + (g - 1.0) / (2.0 * g * self.rho_inf) * self.prandtl * y * (1.0 - y))

    def exact_state(self, x):
        y = np.asarray(x)[:, 1]
        rho = self.gamma * self.p_inf / self.temperature(y)
        v = np.zeros((len(y), 3))
        v[:, 0] = y * np.log1p(y)
        return conserved(rho, v, np.full_like(y, self.p_inf), self.params)

    def source(self, x):
        y = np.asarray(x)[:, 1]
        mu_re = self.params.mu / self.reynolds
        lg = np.log1p(y)
        v1, dv1, ddv1 = y * lg, lg + y / (1.0 + y), (2.0 + y) / (1.0 + y) ** 2
        out = np.zeros((len(y), 5))
        out[:, 1] = -mu_re * ddv1
        out[:, 4] = -mu_re * (ddv1 * v1 + dv1**2 - self.t_inf)
        return out

    def boundary_conditions(self):
        return {lbl: ("dirichlet_state", self.exact_state) for lbl in BOUNDARY_LABELS}


@dataclass
class TgvCase:
    """Taylor-Green vortex initial state, acoustic scaling (cases.py:110-158)."""

    reynolds: float = 100.0
    mach: float = 0.1
    gamma: float = 1.4
    prandtl: float = 0.71
    length: float = 1.0
    rho0: float = 1.0
    params: FlowParams = field(init=False)

    def __post_init__(self):
        self.params = FlowParams(gamma=self.gamma, prandtl=self.prandtl,
                                 reynolds_acoustic=self.reynolds / self.mach, mach_ref=self.mach)

    @property
    def p0(self):
        return 1.0 / self.gamma

    @property
    def v0(self):
        return self.mach

    @property
    def domain(self):
        s = np.pi * self.length
        return (-s, -s, -s), (s, s, s)

    def initial_state(self, x):
        x = np.asarray(x) / self.length
        v0 = self.v0
        v = np.empty((len(x), 3))
        v[:, 0] = v0 * np.sin(x[:, 0]) * np.cos(x[:, 1]) * np.cos(x[:, 2])
        v[:, 1] = -v0 * np.cos(x[:, 0]) * np.sin(x[:, 1]) * np.cos(x[:, 2])
        v[:, 2] = 0.0
        P = self.p0 + (self.rho0 * v0**2 / 16.0) * (np.cos(2 * x[:, 0]) + np.cos(2 * x[:, 1])) * (
            np.cos(2 * x[:, 2]) + 2.0)
        return conserved(self.rho0 * P / self.p0, v, P, self.params)


@dataclass
class CouettePlane2D:
    """C1: steady plane Couette flow, walls at y=0 (fixed) and y=height (moving).

    Acoustic scaling: c_inf = 1 at T_inf = 1 (gamma P = rho T), wall speed
    u_w = mach, both walls at T_w = 1, Re_acoustic = Re/M so that the flow
    Reynolds number is Re.  Exact solution: u = u_w y/H, constant pressure,
    rho = gamma P / T.  In the implemented units
    (gamma P = rho T, e = T/(gamma(gamma-1)), heat flux k_t grad T with
    k_t = gamma mu/((gamma-1) Re Pr)) the energy balance k_t T'' = -mu u'^2/Re
    gives T = T_w + (gamma-1) Pr u_w^2/(2 gamma) eta (1 - eta), eta = y/H.
    """

    reynolds: float = 100.0
    mach: float = 0.15
    gamma: float = 1.4
    prandtl: float = 0.72
    height: float = 1.0
    length: float = 2.0
    t_wall: float = 1.0
    p0: float = 1.0 / 1.4
    params: FlowParams = field(init=False)

    def __post_init__(self):
        self.params = FlowParams(gamma=self.gamma, prandtl=self.prandtl,
                                 reynolds_acoustic=self.reynolds / self.mach, mach_ref=self.mach)

    @property
    def domain(self):
        return (0.0, 0.0), (self.length, self.height)

    @property
    def wall_speed(self):
        return self.mach

    def temperature(self, y):
        eta = np.asarray(y) / self.height
        g = self.gamma
        return self.t_wall + (g - 1.0) * self.prandtl * self.wall_speed**2 / (2.0 * g) * eta * (1.0 - eta)

    def exact_state(self, x):
        y = np.asarray(x)[:, 1]
        T = self.temperature(y)
        rho = self.gamma * self.p0 / T
        v = np.zeros((len(y), 2))
        v[:, 0] = self.wall_speed * y / self.height
        return conserved(rho, v, np.full_like(y, self.p0), self.params)

    def boundary_conditions(self):
        return {"y0": ("isothermal_noslip_wall", self.t_wall),
                "y1": ("isothermal_moving_wall", (self.t_wall, (self.wall_speed, 0.0)))}


@dataclass
class UniformFlow2D:
    """C2 state: rho=1, v=(1, 0.3), P = 1/(gamma M^2); flow scaling (Re_flow = Re)."""

    reynolds: float = 100.0
    mach: float = 0.2
    gamma: float = 1.4
    prandtl: float = 0.72
    velocity: tuple = (1.0, 0.3)
    params: FlowParams = field(init=False)

    def __post_init__(self):
        self.params = FlowParams(gamma=self.gamma, prandtl=self.prandtl, reynolds_acoustic=self.reynolds,
                                 mach_ref=self.mach, reynolds_flow=self.reynolds)

    @property
    def pressure(self):
        return 1.0 / (self.gamma * self.mach**2)

    @property
    def domain(self):
        return (0.0, 0.0), (1.0, 1.0)

    def state(self, x):
        n = len(np.asarray(x))
        return conserved(np.ones(n), np.tile(np.asarray(self.velocity, float), (n, 1)),
                         np.full(n, self.pressure), self.params)


@dataclass
class SphereCase:
    """C4: free stream |v| = M along x past a unit-diameter sphere at Re (based on the
    diameter).  Acoustic scaling as TgvCase (rho = 1, c = 1, P = 1/gamma,
    Re_acoustic = Re/M); BASELINE does not give Pr, 0.72 as C1/C2."""

    reynolds: float = 100.0
    mach: float = 0.2
    gamma: float = 1.4
    prandtl: float = 0.72
    params: FlowParams = field(init=False)

    def __post_init__(self):
        self.params = FlowParams(gamma=self.gamma, prandtl=self.prandtl,
                                 reynolds_acoustic=self.reynolds / self.mach, mach_ref=self.mach)

    def freestream(self, x):
        n = len(np.asarray(x))
        v = np.zeros((n, 3))
        v[:, 0] = self.mach
        return conserved(np.ones(n), v, np.full(n, 1.0 / self.gamma), self.params)

    def boundary_conditions(self):
        return {"sphere": ("adiabatic_noslip_wall", None), "farfield": ("dirichlet_state", self.freestream)}
