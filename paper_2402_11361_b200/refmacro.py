"""Reference macro-element tables for simplicial macro-elements in 2D and 3D.

Host-side setup (built once per (dim, m, p) and uploaded to the device).  A
macro-simplex is split uniformly into m^dim sub-simplices carrying a
continuous piecewise-P_p space whose nodes form the principal lattice of
degree N = m*p.  Faces carry the continuous piecewise-P_p space of the
(dim-1)-simplex split into m^(dim-1) pieces.

Follows ``/root/reference/pkg/src/macrohdg/basis.py`` (RefMacro
basis.py:354-480, quadrature_rule basis.py:173-209, subdivide_macro_tet
basis.py:302-328, _tri_subdivision basis.py:331-339) and generalises it to
dim 2 (triangular macro-elements with edge faces), which the reference lacks.
Node, sub-element and quadrature-point orderings are the reference's, so that
3D tables compare entry-for-entry with it.

The nodal basis is built from monomials instead of the reference's Dubiner
modes; for p <= 3 the Vandermonde system is well conditioned and the tables
agree with the reference to rounding.
"""

from __future__ import annotations

import itertools
from functools import lru_cache
from math import comb, factorial

import numpy as np
from scipy.special import roots_jacobi, roots_legendre

# unit-simplex vertices; local face f is opposite local vertex f, its corners
# listed in ascending local-vertex order (basis.py:21-25 for dim 3)
SIMPLEX_VERTICES = {
    1: np.array([[0.0], [1.0]]),
    2: np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0]]),
    3: np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 1.0]]),
}
FACE_CORNERS = {
    2: ((1, 2), (0, 2), (0, 1)),
    3: ((1, 2, 3), (0, 2, 3), (0, 1, 3), (0, 1, 2)),
}


def multi_indices(dim: int, n: int) -> np.ndarray:
    """All (i_1..i_dim) >= 0 with sum <= n, sorted lexicographically."""
    out = [c for c in itertools.product(range(n + 1), repeat=dim) if sum(c) <= n]
    out.sort()
    return np.array(out, dtype=np.int64).reshape(len(out), dim)


def lattice_size(dim: int, n: int) -> int:
    return comb(n + dim, dim)


# ---------------------------------------------------------------------------
# nodal Lagrange basis on the unit simplex (monomial Vandermonde)
# ---------------------------------------------------------------------------


class NodalBasis:
    """Degree-p Lagrange basis on the unit dim-simplex, equispaced lattice nodes."""

    def __init__(self, dim: int, p: int):
        if dim not in (1, 2, 3) or p < 1:
            raise ValueError("NodalBasis needs dim in (1,2,3) and p >= 1")
        self.dim, self.p = dim, p
        self.multi_indices = multi_indices(dim, p)
        self.nodes = self.multi_indices.astype(float) / p
        self.n_basis = len(self.nodes)
        self._exps = multi_indices(dim, p)
        self._coef = np.linalg.inv(self._mono(self.nodes))

    def _mono(self, x):
        x = np.atleast_2d(x)
        out = np.ones((x.shape[0], len(self._exps)))
        for c, e in enumerate(self._exps):
            for d in range(self.dim):
                if e[d]:
                    out[:, c] *= x[:, d] ** e[d]
        return out

    def _mono_grad(self, x):
        x = np.atleast_2d(x)
        out = np.zeros((x.shape[0], len(self._exps), self.dim))
        for c, e in enumerate(self._exps):
            for r in range(self.dim):
                if e[r] == 0:
                    continue
                term = np.full(x.shape[0], float(e[r]))
                for d in range(self.dim):
                    pw = e[d] - 1 if d == r else e[d]
                    if pw:
                        term = term * x[:, d] ** pw
                out[:, c, r] = term
        return out

    def eval(self, x) -> np.ndarray:
        return self._mono(x) @ self._coef

    def eval_grad(self, x) -> np.ndarray:
        return np.einsum("qcr,cn->qnr", self._mono_grad(x), self._coef)


# ---------------------------------------------------------------------------
# collapsed Gauss-Jacobi quadrature (basis.py:173-209), plus the 1D rule
# ---------------------------------------------------------------------------


@lru_cache(maxsize=None)
def simplex_quadrature(dim: int, order: int):
    """Points/weights on the unit simplex, exact to `order`; weights sum to 1/dim!."""
    if order < 1 or order > 40:
        raise ValueError(f"quadrature order {order} outside [1, 40]")
    n = (order + 2) // 2
    xa, wa = roots_legendre(n)
    if dim == 1:
        return ((xa + 1.0) / 2.0)[:, None], wa / 2.0
    xb, wb = roots_jacobi(n, 1.0, 0.0)
    if dim == 2:
        A, B = np.meshgrid(xa, xb, indexing="ij")
        WA, WB = np.meshgrid(wa, wb, indexing="ij")
        r = 0.5 * (1.0 + A) * (1.0 - B) - 1.0
        pts = np.stack([(r + 1.0) / 2.0, (B + 1.0) / 2.0], axis=-1).reshape(-1, 2)
        return pts, (WA * WB).reshape(-1) / 8.0
    xc, wc = roots_jacobi(n, 2.0, 0.0)
    A, B, C = np.meshgrid(xa, xb, xc, indexing="ij")
    WA, WB, WC = np.meshgrid(wa, wb, wc, indexing="ij")
    r = 0.25 * (1.0 + A) * (1.0 - B) * (1.0 - C) - 1.0
    s = 0.5 * (1.0 + B) * (1.0 - C) - 1.0
    pts = np.stack([(r + 1.0) / 2.0, (s + 1.0) / 2.0, (C + 1.0) / 2.0], axis=-1)
    return pts.reshape(-1, 3), (WA * WB * WC).reshape(-1) / 64.0


# ---------------------------------------------------------------------------
# uniform subdivisions (integer vertices on the degree-m lattice)
# ---------------------------------------------------------------------------


def subdivide_simplex(dim: int, m: int) -> np.ndarray:
    """m^dim positively oriented sub-simplices tiling the unit simplex.

    dim 3: Freudenthal/Kuhn split of the cube grid restricted to x>=y>=z and
    sheared onto the unit tet (basis.py:302-328).  dim 2: the row-by-row
    split of basis.py:331-339.  dim 1: m segments.
    """
    if m < 1:
        raise ValueError("m must be >= 1")
    if dim == 1:
        return np.array([[[i], [i + 1]] for i in range(m)], dtype=np.int64)
    if dim == 2:
        tris = []
        for i in range(m):
            for j in range(m - i):
                tris.append([[i, j], [i + 1, j], [i, j + 1]])
                if i + j < m - 1:
                    tris.append([[i + 1, j], [i + 1, j + 1], [i, j + 1]])
        return np.array(tris, dtype=np.int64)
    shear = np.array([[1, -1, 0], [0, 1, -1], [0, 0, 1]], dtype=np.int64)
    out = []
    for cell in itertools.product(range(m), repeat=3):
        base = np.array(cell, dtype=np.int64)
        for perm in itertools.permutations(range(3)):
            path = [base.copy()]
            for ax in perm:
                nxt = path[-1].copy()
                nxt[ax] += 1
                path.append(nxt)
            if not all(v[0] >= v[1] >= v[2] for v in path):
                continue
            std = np.array(path) @ shear.T
            if np.linalg.det((std[1:] - std[0]).astype(float)) < 0:
                std = std[[0, 2, 1, 3]]
            out.append(std)
    out = np.array(out, dtype=np.int64)
    assert len(out) == m**3
    return out


def _lattice_node(verts_p: np.ndarray, alpha: np.ndarray, p: int) -> np.ndarray:
    """Integer coords (x p) of local node alpha of a sub-simplex with vertices*p."""
    node = (p - alpha.sum()) * verts_p[0]
    for i, a in enumerate(alpha):
        node = node + a * verts_p[i + 1]
    return node


class RefMacro:
    """Tables shared by all affine macro-elements of a given (dim, m, p).

    Attribute names follow the reference RefMacro (basis.py:354-480):
    n_vol (L), n_face_lattice (Lf), n_sub, n_loc, n_quad, sub_conn, phi_vol,
    grad_ref, w_ref, x_ref, mass, mass_inv, weak_deriv, mass_inv_weak_deriv,
    n_loc_face, n_quad_face, phi_face, tri_sub/n_tri (face sub-elements),
    tri_conn, face_quad_bary, w_face_ref, face_mass, face_vol_nodes.
    """

    def __init__(self, dim: int, m: int, p: int, quad_order: int | None = None):
        if dim not in (2, 3):
            raise ValueError("dim must be 2 or 3")
        if m < 1 or p < 1:
            raise ValueError("m and p must be >= 1")
        self.dim, self.m, self.p = dim, m, p
        N = self.n_lattice = m * p
        order = self.quad_order = quad_order if quad_order is not None else 2 * p + 1

        # volume lattice and sub-element connectivity
        self.vol_multi = multi_indices(dim, N)
        self.vol_coords = self.vol_multi.astype(float) / N
        self.n_vol = len(self.vol_multi)
        vol_id = {tuple(r): i for i, r in enumerate(self.vol_multi)}
        self.subtet_verts = subdivide_simplex(dim, m)
        self.n_sub = len(self.subtet_verts)
        vb = NodalBasis(dim, p)
        self.n_loc = vb.n_basis
        self.sub_conn = np.array(
            [
                [vol_id[tuple(_lattice_node(sv * p, al, p) // p)] for al in vb.multi_indices]
                for sv in self.subtet_verts
            ],
            dtype=np.int64,
        )

        # volume quadrature per sub-element
        qp, qw = simplex_quadrature(dim, order)
        self.n_quad = len(qw)
        self.phi_vol = vb.eval(qp)
        dphi = vb.eval_grad(qp)
        self.grad_ref = np.empty((self.n_sub, self.n_quad, self.n_loc, dim))
        self.x_ref = np.empty((self.n_sub, self.n_quad, dim))
        self.w_ref = np.empty((self.n_sub, self.n_quad))
        for K, sv in enumerate(self.subtet_verts):
            v = sv.astype(float) / m
            B = (v[1:] - v[0]).T
            self.grad_ref[K] = np.einsum("qnm,ml->qnl", dphi, np.linalg.inv(B))
            self.x_ref[K] = v[0] + qp @ B.T
            self.w_ref[K] = qw * abs(np.linalg.det(B))

        # reference mass and weak derivative, D[l][i, j] = int phi_j d_l phi_i
        L = self.n_vol
        self.mass = np.zeros((L, L))
        self.weak_deriv = np.zeros((dim, L, L))
        for K in range(self.n_sub):
            ix = np.ix_(self.sub_conn[K], self.sub_conn[K])
            self.mass[ix] += np.einsum("q,qa,qb->ab", self.w_ref[K], self.phi_vol, self.phi_vol)
            for l in range(dim):
                self.weak_deriv[l][ix] += np.einsum(
                    "q,qa,qb->ab", self.w_ref[K], self.grad_ref[K][:, :, l], self.phi_vol
                )
        self.mass_inv = np.linalg.inv(self.mass)
        self.mass_inv_weak_deriv = np.einsum("ij,ljk->lik", self.mass_inv, self.weak_deriv)

        # face lattice, face sub-elements and their quadrature
        fdim = dim - 1
        self.face_multi = multi_indices(fdim, N)
        self.n_face_lattice = len(self.face_multi)
        face_id = {tuple(r): i for i, r in enumerate(self.face_multi)}
        fb = NodalBasis(fdim, p)
        self.n_loc_face = fb.n_basis
        fqp, fqw = simplex_quadrature(fdim, order)
        self.n_quad_face = len(fqw)
        self.phi_face = fb.eval(fqp)
        self.tri_sub = subdivide_simplex(fdim, m)
        self.n_tri = len(self.tri_sub)
        self.tri_conn = np.array(
            [
                [face_id[tuple(_lattice_node(tv * p, al, p) // p)] for al in fb.multi_indices]
                for tv in self.tri_sub
            ],
            dtype=np.int64,
        )
        self.face_quad_bary = np.empty((self.n_tri, self.n_quad_face, dim))
        self.w_face_ref = np.empty((self.n_tri, self.n_quad_face))
        for T, tv in enumerate(self.tri_sub):
            v = tv.astype(float) / m
            B = (v[1:] - v[0]).T
            xf = v[0] + fqp @ B.T
            self.face_quad_bary[T, :, 1:] = xf
            self.face_quad_bary[T, :, 0] = 1.0 - xf.sum(axis=1)
            self.w_face_ref[T] = fqw * abs(np.linalg.det(B))
        Lf = self.n_face_lattice
        self.face_mass = np.zeros((Lf, Lf))
        for T in range(self.n_tri):
            ix = np.ix_(self.tri_conn[T], self.tri_conn[T])
            self.face_mass[ix] += np.einsum(
                "q,qa,qb->ab", self.w_face_ref[T], self.phi_face, self.phi_face
            )

        # volume nodes on each local face, in face-lattice order
        corners = (SIMPLEX_VERTICES[dim] * N).astype(np.int64)
        self.n_faces_local = dim + 1
        self.face_vol_nodes = np.empty((dim + 1, Lf), dtype=np.int64)
        for lf, fc in enumerate(FACE_CORNERS[dim]):
            cc = corners[list(fc)]
            for g, al in enumerate(self.face_multi):
                self.face_vol_nodes[lf, g] = vol_id[tuple(_lattice_node(cc, al, N) // N)]

    @property
    def face_measure_factor(self) -> float:
        """(dim-1)!: maps w_face_ref (summing to 1/(dim-1)!) to the face measure."""
        return float(factorial(self.dim - 1))


@lru_cache(maxsize=None)
def ref_macro(dim: int, m: int, p: int, quad_order: int | None = None) -> RefMacro:
    return RefMacro(dim, m, p, quad_order)
