"""Legacy ASCII VTK output of the sub-element mesh and nodal fields.

The reference declares `mesh.write_vtk_mesh` (mesh.py:375-379) on top of an
`io_utils.write_vtk` that is not shipped, and SPEC.md asks for "legacy ASCII VTK
unstructured grid (sub-tet level)" with point data rho, v, P.
This is that writer: one linear simplex per sub-element of every macro (the
sub-element's d+1 corner lattice nodes), points = the macro's volume lattice
nodes (duplicated per macro, so fields stay discontinuous as the discretization),
point data from the conserved state u (n_mac, L, ns) in the reference layout.
Host numpy; for inspection, not on the hot path.
"""

from __future__ import annotations

import numpy as np

VTK_TRIANGLE, VTK_TETRA = 5, 10


def _corner_nodes(rm) -> np.ndarray:
    """(n_sub, d+1) lattice node index of every sub-element corner."""
    coords = rm.vol_coords
    out = np.empty(rm.subtet_verts.shape[:2], dtype=np.int64)
    for K, verts in enumerate(rm.subtet_verts):
        for i, v in enumerate(np.asarray(verts, dtype=float) / rm.m):
            out[K, i] = int(np.argmin(np.abs(coords - v).sum(axis=1)))
    return out


def primitives(u: np.ndarray, gamma: float):
    """rho, v, P from conserved nodal values (physics.py conventions)."""
    d = u.shape[-1] - 2
    rho = u[..., 0]
    v = u[..., 1: 1 + d] / rho[..., None]
    P = (gamma - 1.0) * (u[..., 1 + d] - 0.5 * rho * (v * v).sum(-1))
    return rho, v, P


def write_vtk(disc, path, u=None) -> None:
    """Write `disc`'s sub-element mesh (and, with u, rho / velocity / pressure at the
    lattice nodes) to `path` as legacy VTK 3.0 ASCII."""
    rm, d = disc.rm, disc.dim
    X = disc.node_coords()  # (n_mac, L, d)
    M, L = X.shape[:2]
    corners = _corner_nodes(rm)
    pts = X.reshape(-1, d)
    if d == 2:
        pts = np.column_stack([pts, np.zeros(len(pts))])
    cells = (np.arange(M)[:, None, None] * L + corners[None]).reshape(-1, d + 1)
    ctype = VTK_TETRA if d == 3 else VTK_TRIANGLE
    with open(path, "w") as fh:
        fh.write("# vtk DataFile Version 3.0\nmacro-element HDG sub-element mesh\nASCII\nDATASET UNSTRUCTURED_GRID\n")
        fh.write(f"POINTS {len(pts)} double\n")
        np.savetxt(fh, pts, fmt="%.17g")
        fh.write(f"CELLS {len(cells)} {len(cells) * (d + 2)}\n")
        np.savetxt(fh, np.column_stack([np.full(len(cells), d + 1), cells]), fmt="%d")
        fh.write(f"CELL_TYPES {len(cells)}\n")
        np.savetxt(fh, np.full(len(cells), ctype), fmt="%d")
        if u is not None:
            u = np.asarray(u.detach().cpu() if hasattr(u, "detach") else u, dtype=float).reshape(M, L, d + 2)
            rho, v, P = primitives(u, disc.params.gamma)
            fh.write(f"POINT_DATA {len(pts)}\n")
            for name, arr in (("rho", rho), ("P", P)):
                fh.write(f"SCALARS {name} double 1\nLOOKUP_TABLE default\n")
                np.savetxt(fh, arr.reshape(-1), fmt="%.17g")
            vv = v.reshape(-1, d)
            if d == 2:
                vv = np.column_stack([vv, np.zeros(len(vv))])
            fh.write("VECTORS velocity double\n")
            np.savetxt(fh, vv, fmt="%.17g")


def write_vtk_mesh(disc, path) -> None:
    """mesh.py:375-379 of the reference: the sub-element mesh alone."""
    write_vtk(disc, path)
