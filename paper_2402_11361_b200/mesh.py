"""Macro-element simplicial meshes of boxes (2D triangles, 3D tetrahedra).

Host-side setup, not accelerated.  Follows ``mesh.py`` of the reference
(MacroMesh mesh.py:30-108, _build_faces mesh.py:132-225, build_cube_mesh
mesh.py:228-298, count_dofs mesh.py:361-372) and adds the 2D box mesh the
BASELINE 2D configs need (squares split along the SW->NE diagonal).  The face
skeleton is ordered exactly as the reference orders it (sorted vertex-id keys,
max-side periodic faces folded into their min-side partner), so 3D trace
vectors are index-compatible with the reference.
"""

from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

from .refmacro import FACE_CORNERS, lattice_size

INTERIOR = 0
BOUNDARY = 1
PERIODIC = 2

# box planes (codes 0-5, the reference's labels) and the O-grid's two spheres (6, 7)
BOUNDARY_LABELS = ("x0", "x1", "y0", "y1", "z0", "z1", "sphere", "farfield")


@dataclass
class MacroMesh:
    """Conforming macro-simplex mesh plus its face skeleton.

    corner_map[f, side, r] is the position, in that side's local face-corner
    order, of the face's canonical corner r (side 0 defines the canonical
    order).  Boundary faces have macro -1 on side 1.
    """

    vertices: np.ndarray
    macro_tets: np.ndarray  # (n_mac, dim+1) vertex ids
    m: int
    face_macros: np.ndarray
    face_locals: np.ndarray
    face_kind: np.ndarray
    face_label: np.ndarray
    corner_map: np.ndarray
    periodic_offset: np.ndarray
    faces_of_macro: np.ndarray = field(init=False)
    sides_of_macro: np.ndarray = field(init=False)
    jac: np.ndarray = field(init=False)
    inv_jac: np.ndarray = field(init=False)
    det: np.ndarray = field(init=False)
    normals: np.ndarray = field(init=False)
    areas: np.ndarray = field(init=False)

    def __post_init__(self):
        nm, nv = self.macro_tets.shape
        d = nv - 1
        self.dim = d
        self.faces_of_macro = np.full((nm, nv), -1, dtype=np.int64)
        self.sides_of_macro = np.full((nm, nv), -1, dtype=np.int64)
        for side in range(2):
            ok = self.face_macros[:, side] >= 0
            f_ids = np.nonzero(ok)[0]
            self.faces_of_macro[self.face_macros[ok, side], self.face_locals[ok, side]] = f_ids
            self.sides_of_macro[self.face_macros[ok, side], self.face_locals[ok, side]] = side
        if np.any(self.faces_of_macro < 0):
            raise AssertionError("incomplete face skeleton")

        X = self.vertices[self.macro_tets]  # (nm, d+1, d)
        jac = np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1))
        det = np.linalg.det(jac)
        if np.any(det <= 0):
            raise AssertionError("macro-element with non-positive jacobian determinant")
        self.jac, self.inv_jac, self.det = jac, np.linalg.inv(jac), det

        normals = np.empty((nm, nv, d))
        areas = np.empty((nm, nv))
        cen = X.mean(axis=1)
        for lf, fc in enumerate(FACE_CORNERS[d]):
            P = X[:, list(fc)]
            if d == 3:
                nvec = 0.5 * np.cross(P[:, 1] - P[:, 0], P[:, 2] - P[:, 0])
            else:
                t = P[:, 1] - P[:, 0]
                nvec = np.stack([t[:, 1], -t[:, 0]], axis=-1)
            a = np.linalg.norm(nvec, axis=1)
            nu = nvec / a[:, None]
            flip = np.einsum("ij,ij->i", nu, P.mean(axis=1) - cen) < 0
            nu[flip] *= -1.0
            normals[:, lf], areas[:, lf] = nu, a
        self.normals, self.areas = normals, areas

    @property
    def n_macro(self) -> int:
        return len(self.macro_tets)

    @property
    def n_faces(self) -> int:
        return len(self.face_macros)

    def macro_volumes(self) -> np.ndarray:
        return self.det / (6.0 if self.dim == 3 else 2.0)


def _orient_positive(tets, vertices):
    X = vertices[tets]
    det = np.linalg.det(np.transpose(X[:, 1:] - X[:, :1], (0, 2, 1)))
    tets = tets.copy()
    flip = det < 0
    tets[flip, 1], tets[flip, 2] = tets[flip, 2].copy(), tets[flip, 1].copy()
    return tets


def build_faces(vertices, tets, lo, hi, periodic, tol, classify=None):
    """Face skeleton in the reference's order (mesh.py:132-225), any dim.
    classify(face vertex coords (d, d)) -> label code replaces the box-plane
    tags (mesh.py:144-151) for meshes that are not boxes."""
    d = tets.shape[1] - 1
    corners = FACE_CORNERS[d]
    nm = len(tets)
    # (nm, d+1, d) face vertex gids in local corner order
    fg = tets[:, np.array(corners)]
    flat = fg.reshape(nm * (d + 1), d)
    keys = np.sort(flat, axis=1)
    uniq, inv, counts = np.unique(keys, axis=0, return_inverse=True, return_counts=True)
    inv = inv.reshape(-1)
    if np.any(counts > 2):
        raise AssertionError("face with more than two incidences")
    order = np.argsort(inv, kind="stable")
    start = np.concatenate([[0], np.cumsum(counts)])

    qscale = tol * 10
    vkey = {tuple(np.round(v / qscale).astype(np.int64)): i for i, v in enumerate(vertices)}

    def find_vertex(pos):
        base = np.round(pos / qscale).astype(np.int64)
        for dk in itertools.product((0, -1, 1), repeat=len(pos)):
            k = tuple(base + np.array(dk))
            if k in vkey:
                return vkey[k]
        raise KeyError(f"no vertex at {pos}")

    def bcode(gids):
        P = vertices[list(gids)]
        for ax in range(d):
            if np.all(np.abs(P[:, ax] - lo[ax]) < tol):
                return 2 * ax
            if np.all(np.abs(P[:, ax] - hi[ax]) < tol):
                return 2 * ax + 1
        return -1

    key_index = {tuple(k): i for i, k in enumerate(uniq)} if np.any(periodic) else None
    recs = []
    for u in range(len(uniq)):
        incs = order[start[u] : start[u + 1]]
        if len(incs) == 2:
            i0, i1 = incs
            g0, g1 = tuple(flat[i0]), tuple(flat[i1])
            recs.append(((i0 // (d + 1), i1 // (d + 1)), (i0 % (d + 1), i1 % (d + 1)),
                         INTERIOR, -1, g0, g1, np.zeros(d)))
            continue
        i0 = incs[0]
        g0 = tuple(flat[i0])
        code = bcode(g0) if classify is None else int(classify(vertices[list(g0)]))
        if code < 0:
            raise AssertionError("single-incidence face not on the box boundary")
        ax = code // 2
        if classify is not None or not periodic[ax]:
            recs.append(((i0 // (d + 1), -1), (i0 % (d + 1), -1), BOUNDARY, code, g0, None,
                         np.zeros(d)))
            continue
        if code % 2 == 1:
            continue  # folded into the min-side partner
        off = np.zeros(d)
        off[ax] = hi[ax] - lo[ax]
        partner = tuple(find_vertex(vertices[g] + off) for g in g0)
        pk = key_index.get(tuple(sorted(partner)))
        if pk is None or counts[pk] != 1:
            raise AssertionError("periodic partner face not found")
        i1 = order[start[pk]]
        g1 = tuple(flat[i1])
        recs.append(((i0 // (d + 1), i1 // (d + 1)), (i0 % (d + 1), i1 % (d + 1)),
                     PERIODIC, -1, partner, g1, -off))

    nf = len(recs)
    face_macros = np.full((nf, 2), -1, dtype=np.int64)
    face_locals = np.full((nf, 2), -1, dtype=np.int64)
    face_kind = np.zeros(nf, dtype=np.int64)
    face_label = np.full(nf, -1, dtype=np.int64)
    corner_map = np.zeros((nf, 2, d), dtype=np.int64)
    offs = np.zeros((nf, d))
    ident = np.arange(d)
    for f, (macs, locs, kind, label, canon1, g1, off) in enumerate(recs):
        face_macros[f], face_locals[f] = macs, locs
        face_kind[f], face_label[f], offs[f] = kind, label, off
        corner_map[f, 0] = ident
        if g1 is not None:
            corner_map[f, 1] = [g1.index(g) for g in canon1]
    return face_macros, face_locals, face_kind, face_label, corner_map, offs


def _kuhn_cell_tets():
    out = []
    for perm in itertools.permutations(range(3)):
        path = [np.zeros(3, dtype=np.int64)]
        for ax in perm:
            nxt = path[-1].copy()
            nxt[ax] += 1
            path.append(nxt)
        out.append(np.array(path))
    return out


def build_cube_mesh(domain, n_ele_1d: int, m: int, periodic=(False, False, False),
                    split: str = "kuhn") -> MacroMesh:
    """Structured 3D macro-tet mesh of a box: n^3 cells x 6 Kuhn tets (mesh.py:228-298)."""
    if split != "kuhn":
        raise ValueError("only the kuhn split is provided")
    if n_ele_1d < 1 or m < 1:
        raise ValueError("n_ele_1d and m must be >= 1")
    lo, hi = np.asarray(domain[0], float), np.asarray(domain[1], float)
    if np.any(hi <= lo):
        raise ValueError("domain must have positive extent along every axis")
    n = n_ele_1d
    h = (hi - lo) / n
    ids = np.arange((n + 1) ** 3).reshape(n + 1, n + 1, n + 1)
    g = [lo[a] + h[a] * np.arange(n + 1) for a in range(3)]
    X, Y, Z = np.meshgrid(*g, indexing="ij")
    vertices = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=-1)
    cells = np.array(list(itertools.product(range(n), repeat=3)), dtype=np.int64)
    tets = []
    for off in _kuhn_cell_tets():
        c = cells[:, None, :] + off[None, :, :]  # (ncell, 4, 3)
        tets.append(ids[c[..., 0], c[..., 1], c[..., 2]])
    tets = np.stack(tets, axis=1).reshape(-1, 4)  # cell-major, 6 tets per cell
    tets = _orient_positive(tets, vertices)
    faces = build_faces(vertices, tets, lo, hi, periodic, float(np.min(h)) * 1e-8)
    return MacroMesh(vertices, tets, m, *faces)


def build_square_mesh(domain, n_cells, m: int, periodic=(False, False)) -> MacroMesh:
    """Structured 2D macro-triangle mesh: nx x ny squares, each split along its
    SW->NE diagonal into (v00, v10, v11) and (v00, v11, v01); cells i-major."""
    lo, hi = np.asarray(domain[0], float), np.asarray(domain[1], float)
    nx, ny = (n_cells, n_cells) if np.isscalar(n_cells) else tuple(n_cells)
    if nx < 1 or ny < 1 or m < 1:
        raise ValueError("cell counts and m must be >= 1")
    if np.any(hi <= lo):
        raise ValueError("domain must have positive extent along every axis")
    hx, hy = (hi - lo) / np.array([nx, ny])
    ids = np.arange((nx + 1) * (ny + 1)).reshape(nx + 1, ny + 1)
    X, Y = np.meshgrid(lo[0] + hx * np.arange(nx + 1), lo[1] + hy * np.arange(ny + 1),
                       indexing="ij")
    vertices = np.stack([X.ravel(), Y.ravel()], axis=-1)
    I, J = np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij")
    I, J = I.ravel(), J.ravel()
    v00, v10, v01, v11 = ids[I, J], ids[I + 1, J], ids[I, J + 1], ids[I + 1, J + 1]
    tris = np.stack([np.stack([v00, v10, v11], -1), np.stack([v00, v11, v01], -1)], axis=1)
    tris = _orient_positive(tris.reshape(-1, 3), vertices)
    faces = build_faces(vertices, tris, lo, hi, tuple(periodic), float(min(hx, hy)) * 1e-8)
    return MacroMesh(vertices, tris, m, *faces)


def build_sphere_ogrid_mesh(n_r: int, n_theta: int, n_phi: int, m: int, r_in: float = 0.5,
                            r_out: float = 20.0, grading: float = 1.15) -> MacroMesh:
    """O-grid around a sphere (BASELINE config 4; the reference meshes boxes only,
    mesh.py:144-151): n_r radial shells geometrically graded (ratio `grading`) from
    r_in to r_out, x n_theta polar x n_phi azimuthal cells in spherical coordinates,
    each cell split into 6 Kuhn tets in (r, theta, phi) index space, as
    build_cube_mesh does (mesh.py:263-266); cells r-major, so contiguous macro
    slabs are radial shells.

    Poles: the cells touching the polar axis are wedges (their theta = 0 or pi
    corners coincide for every phi).  The axis vertices are shared and the Kuhn
    tets with a repeated vertex (three of the six in a wedge cell, zero volume)
    are dropped; the other three tile the wedge conformingly, since a dropped
    tet's two non-degenerate faces coincide and become the interface of the two
    neighbouring tets.  phi wraps through the vertex numbering (no periodic faces).
    Boundary labels: "sphere" (r = r_in) and "farfield" (r = r_out)."""
    if n_r < 1 or n_theta < 2 or n_phi < 3 or m < 1:
        raise ValueError("need n_r >= 1, n_theta >= 2, n_phi >= 3, m >= 1")
    if not (0.0 < r_in < r_out) or grading <= 0.0:
        raise ValueError("need 0 < r_in < r_out and grading > 0")
    w = grading ** np.arange(n_r)
    r = r_in + (r_out - r_in) * np.concatenate([[0.0], np.cumsum(w)]) / np.sum(w)
    th = np.pi * np.arange(n_theta + 1) / n_theta
    ph = 2.0 * np.pi * np.arange(n_phi) / n_phi
    # vertex ids: interior theta rings (i, j = 1..n_theta-1, k) then the two axis points per radius
    nt_in = n_theta - 1
    ring = np.arange((n_r + 1) * nt_in * n_phi).reshape(n_r + 1, nt_in, n_phi)
    north = ring.size + np.arange(n_r + 1)
    south = north[-1] + 1 + np.arange(n_r + 1)
    R, T, P = np.meshgrid(r, th[1:-1], ph, indexing="ij")
    xyz = np.stack([R * np.sin(T) * np.cos(P), R * np.sin(T) * np.sin(P), R * np.cos(T)], -1).reshape(-1, 3)
    axis = lambda z: np.stack([np.zeros_like(r), np.zeros_like(r), z * r], -1)
    vertices = np.concatenate([xyz, axis(1.0), axis(-1.0)])

    def vid(i, j, k):
        k = k % n_phi
        return np.where(j == 0, north[i], np.where(j == n_theta, south[i], ring[i, np.clip(j - 1, 0, nt_in - 1), k]))

    cells = np.array(list(itertools.product(range(n_r), range(n_theta), range(n_phi))), dtype=np.int64)
    tets = []
    for off in _kuhn_cell_tets():
        c = cells[:, None, :] + off[None, :, :]
        tets.append(vid(c[..., 0], c[..., 1], c[..., 2]))
    tets = np.stack(tets, axis=1).reshape(-1, 4)  # cell-major, 6 Kuhn tets per cell
    srt = np.sort(tets, axis=1)
    tets = tets[np.all(srt[:, 1:] != srt[:, :-1], axis=1)]
    tets = _orient_positive(tets, vertices)
    tol = 1e-8 * float(r[1] - r[0])

    def classify(P):
        rr = np.linalg.norm(P, axis=1)
        if np.all(np.abs(rr - r_in) < tol * 10):
            return BOUNDARY_LABELS.index("sphere")
        if np.all(np.abs(rr - r_out) < tol * 1e3):
            return BOUNDARY_LABELS.index("farfield")
        return -1

    lo, hi = vertices.min(axis=0), vertices.max(axis=0)
    faces = build_faces(vertices, tets, lo, hi, (False, False, False), tol, classify=classify)
    return MacroMesh(vertices, tets, m, *faces)


def count_dofs(mesh: MacroMesh, p: int, n_s: int | None = None):
    """(total local dofs, global trace dofs, local dofs per macro) (mesh.py:361-372)."""
    d = mesh.dim
    return count_dofs_from_counts(mesh.n_macro, mesh.n_faces, mesh.m, p, n_s or d + 2, d)


def count_dofs_from_counts(n_macro, n_faces, m, p, n_s=5, dim=3):
    if p < 1:
        raise ValueError("p must be >= 1")
    per = n_s * (dim + 1) * lattice_size(dim, m * p)
    return n_macro * per, n_s * n_faces * lattice_size(dim - 1, m * p), per
