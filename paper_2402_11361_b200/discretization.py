"""Discretization: mesh + reference tables + trace layout + boundary data.

Host-side setup mirroring ``Discretization`` of the reference
(assembly.py:99-290): same attribute names and layouts (volume dof
node*ns+s, gradient dof (l*L+node)*ns+s, trace dof (f*Lf+g)*ns+s, local
trace (mac, lf, g, s) with the side-1 corner permutation baked into
`gather`, assembly.py:159-179).  Everything here is numpy and runs once; the
device copy of these tables is built lazily by `device.DeviceDisc` the first
time a GPU operation needs it.
"""

from __future__ import annotations

from typing import Callable

import numpy as np

from .mesh import BOUNDARY, BOUNDARY_LABELS, MacroMesh
from .physics import FlowParams
from .refmacro import FACE_CORNERS, SIMPLEX_VERTICES, ref_macro

DIRICHLET = 1
WALL = 2
# adiabatic no-slip wall (BASELINE config 4; the reference has none, physics.py:201):
# rho_hat = rho, m_hat = 0 as the reference's wall (assembly.py:546-550), and the
# energy row E_hat = E (interior total energy, so T_hat = T and the stabilised heat
# flux through the wall vanishes) in place of the isothermal E_hat = rho_hat e_w
ADIABATIC = 3


class ConfigError(ValueError):
    """Inconsistent case configuration (assembly.py:33)."""


class Discretization:
    def __init__(
        self,
        mesh: MacroMesh,
        p: int,
        params: FlowParams,
        bcs: dict | None = None,
        source: Callable | None = None,
        quad_order: int | None = None,
    ):
        self.mesh = mesh
        self.p = p
        self.params = params
        self.source = source
        self.dim = d = mesh.dim
        self.rm = rm = ref_macro(d, mesh.m, p, quad_order)
        self.ns = d + 2
        self.nf = d + 1
        self.n_mac = mesh.n_macro
        self.L = rm.n_vol
        self.Lf = rm.n_face_lattice
        self.n_trace = mesh.n_faces * self.Lf * self.ns
        self.face_fac = rm.face_measure_factor  # face weights = w_face_ref * fac * area

        self.jac, self.inv_jac, self.det = mesh.jac, mesh.inv_jac, mesh.det
        self.origin = mesh.vertices[mesh.macro_tets[:, 0]]
        self.normals, self.areas = mesh.normals, mesh.areas

        # sub-element diameters (SUPG length scale), assembly.py:130-141
        sv = rm.subtet_verts.astype(float) / mesh.m
        X = self.origin[:, None, None, :] + np.einsum("kvr,mlr->mkvl", sv, self.jac)
        h = np.zeros((self.n_mac, rm.n_sub))
        for i in range(d + 1):
            for j in range(i + 1, d + 1):
                h = np.maximum(h, np.linalg.norm(X[:, :, i] - X[:, :, j], axis=-1))
        self.h_sub = h

        # reference coordinates of face quadrature points per local face
        V = SIMPLEX_VERTICES[d]
        self.face_xref = np.stack(
            [np.einsum("tqr,rl->tql", rm.face_quad_bary, V[list(fc)]) for fc in FACE_CORNERS[d]]
        )
        self.node_xref = rm.vol_coords
        self._build_trace_layout()
        self._resolve_bcs(bcs or {})
        self._device = None

    # ------------------------------------------------------------------
    def _build_trace_layout(self):
        mesh, rm, ns, d = self.mesh, self.rm, self.ns, self.dim
        N = rm.n_lattice
        fm = rm.face_multi  # (Lf, d-1)
        bary = np.column_stack([N - fm.sum(axis=1), fm])  # (Lf, d) w.r.t. own corners
        # lattice id from the trailing d-1 barycentric coordinates
        radix = (N + 1) ** np.arange(d - 2, -1, -1)
        lookup = np.full((N + 1) ** (d - 1), -1, dtype=np.int64)
        lookup[fm @ radix] = np.arange(len(fm))
        f_of = mesh.faces_of_macro
        cm = mesh.corner_map[f_of, mesh.sides_of_macro]  # (n_mac, nf, d)
        # canonical barycentrics of this side's local nodes
        cb = bary[:, cm]  # (Lf, n_mac, nf, d)
        g = np.moveaxis(lookup[cb[..., 1:] @ radix], 0, 2)  # (n_mac, nf, Lf)
        dof = (f_of[:, :, None] * self.Lf + g)[..., None] * ns + np.arange(ns)
        self.gather = dof.reshape(self.n_mac, self.nf, self.Lf * ns)

    def _resolve_bcs(self, bcs):
        mesh, d = self.mesh, self.dim
        self.bc_kind = np.zeros((self.n_mac, self.nf), dtype=np.int64)
        self.bc_label = np.full((self.n_mac, self.nf), -1, dtype=np.int64)
        self.bc_data = {}
        g = self.params.gamma
        for lbl, spec in bcs.items():
            code = BOUNDARY_LABELS.index(lbl)
            kind, data = spec
            if kind == "dirichlet_state":
                self.bc_data[code] = (DIRICHLET, data)
            elif kind == "isothermal_noslip_wall":
                self.bc_data[code] = (WALL, (float(data) / (g * (g - 1.0)), np.zeros(d)))
            elif kind == "isothermal_moving_wall":
                T_w, vel = data
                self.bc_data[code] = (WALL, (float(T_w) / (g * (g - 1.0)),
                                             np.asarray(vel, dtype=float).reshape(d)))
            elif kind == "adiabatic_noslip_wall":
                self.bc_data[code] = (ADIABATIC, None)
            else:
                raise ConfigError(f"unknown boundary kind {kind!r}")
        fk = mesh.face_kind[mesh.faces_of_macro]
        fl = mesh.face_label[mesh.faces_of_macro]
        for mac, lf in zip(*np.nonzero(fk == BOUNDARY)):
            code = int(fl[mac, lf])
            if code not in self.bc_data:
                raise ConfigError(f"no boundary condition for face label {BOUNDARY_LABELS[code]!r}")
            self.bc_kind[mac, lf] = self.bc_data[code][0]
            self.bc_label[mac, lf] = code

    # ------------------------------------------------------------------
    def node_coords(self) -> np.ndarray:
        """Physical coordinates of the volume lattice nodes, (n_mac, L, d)."""
        return self.origin[:, None, :] + np.einsum("ar,mlr->mal", self.node_xref, self.jac)

    def face_quad_coords(self, lf: int, tri: int) -> np.ndarray:
        return self.origin[:, None, :] + np.einsum("qr,mlr->mql", self.face_xref[lf, tri], self.jac)

    def volume_quad_coords(self, K: int) -> np.ndarray:
        return self.origin[:, None, :] + np.einsum("qr,mlr->mql", self.rm.x_ref[K], self.jac)

    def nodal_interpolant(self, state_fn):
        """(u, uhat) numpy arrays: nodal interpolation plus owner-side trace
        interpolation (assembly.py:228-245); the gradient is refreshed
        separately."""
        ns, rm = self.ns, self.rm
        X = self.node_coords()
        u = state_fn(X.reshape(-1, self.dim)).reshape(self.n_mac, self.L, ns)
        uhat = np.zeros(self.n_trace)
        own = self.mesh.sides_of_macro == 0
        for lf in range(self.nf):
            macs = np.nonzero(own[:, lf])[0]
            if len(macs) == 0:
                continue
            xf = X[macs][:, rm.face_vol_nodes[lf]]
            vals = state_fn(xf.reshape(-1, self.dim)).reshape(len(macs), self.Lf * ns)
            uhat[self.gather[macs, lf]] = vals
        return u, uhat

    def owner_trace_from_nodes(self, u: np.ndarray) -> np.ndarray:
        """Trace vector copied from the owner side's face volume nodes."""
        uhat = np.zeros(self.n_trace)
        own = self.mesh.sides_of_macro == 0
        for lf in range(self.nf):
            macs = np.nonzero(own[:, lf])[0]
            uhat[self.gather[macs, lf]] = u[macs][:, self.rm.face_vol_nodes[lf]].reshape(len(macs), -1)
        return uhat

    # ------------------------------------------------------------------
    # tables derived for the device path
    def scatter_sources(self) -> np.ndarray:
        """(n_trace, 2) int64 flat indices into the local trace array
        (n_mac*nf*Lf*ns) whose sum is each global trace dof; the lower flat
        index comes first, which is the order np.add.at accumulates in
        (condense.py:48-51).  -1 marks a missing second contribution."""
        flat = self.gather.reshape(-1)
        order = np.argsort(flat, kind="stable")
        counts = np.bincount(flat, minlength=self.n_trace)
        if np.any(counts < 1) or np.any(counts > 2):
            raise AssertionError("trace dof with 0 or >2 local contributions")
        src = np.full((self.n_trace, 2), -1, dtype=np.int64)
        start = np.concatenate([[0], np.cumsum(counts)])
        src[:, 0] = order[start[:-1]]
        two = counts == 2
        src[two, 1] = order[start[:-1][two] + 1]
        return src

    def boundary_tables(self):
        """Per-(macro, local face) boundary data for the device kernels:
        wall_e (n_mac, nf), wall_u (n_mac, nf, d), and the Dirichlet state at
        every face quadrature point (n_mac, nf, n_tri, nqf, ns), zero off the
        Dirichlet faces.  The reference evaluates the same callables inside
        every assembly (assembly.py:542-545); they are time independent."""
        rm, d, ns = self.rm, self.dim, self.ns
        wall_e = np.zeros((self.n_mac, self.nf))
        wall_u = np.zeros((self.n_mac, self.nf, d))
        u_dir = np.zeros((self.n_mac, self.nf, rm.n_tri, rm.n_quad_face, ns))
        for code, (kind, data) in self.bc_data.items():
            sel = self.bc_label == code
            if kind == WALL:
                wall_e[sel] = data[0]
                wall_u[sel] = data[1]
                continue
            if kind == ADIABATIC:
                continue
            for lf in range(self.nf):
                macs = np.nonzero(sel[:, lf])[0]
                if len(macs) == 0:
                    continue
                for T in range(rm.n_tri):
                    x = self.face_quad_coords(lf, T)[macs]
                    u_dir[macs, lf, T] = data(x.reshape(-1, d)).reshape(len(macs), -1, ns)
        return wall_e, wall_u, u_dir

    def source_table(self):
        """Source term at every volume quadrature point, (n_mac, n_sub, nq, ns)."""
        if self.source is None:
            return None
        rm = self.rm
        out = np.empty((self.n_mac, rm.n_sub, rm.n_quad, self.ns))
        for K in range(rm.n_sub):
            x = self.volume_quad_coords(K)
            out[:, K] = self.source(x.reshape(-1, self.dim)).reshape(self.n_mac, rm.n_quad, self.ns)
        return out

    @property
    def device(self):
        """Device-resident copy of the tables (built on first use)."""
        if self._device is None:
            from .device import DeviceDisc

            self._device = DeviceDisc(self)
        return self._device
