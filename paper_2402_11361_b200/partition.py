"""Contiguous macro-slab partition of a macro mesh across ranks (host setup).

The per-macro work is embarrassingly parallel; the only
coupling is the single-valued trace on faces shared by two macros.  Rank r
owns macros [r M / P, (r+1) M / P) (the builders order macros cell-major, so a
slab is a strip of cells), and every face is owned by the rank of its side-0
macro.  The rank's local mesh keeps all faces touching its macros, numbered
[owned faces | ghost faces]; a face whose other side lives on another rank
stays an interior face (its remote side is simply absent locally), so
boundary conditions are untouched.

Exchange plans, per neighbour rank q, list faces in ascending global id on
both sides, so a packed halo needs no index translation:
  * forward halo (trace vectors x): owner sends x on its faces that q holds as
    ghosts; q receives them into its ghost slots;
  * reverse halo (local contributions y): q sends its partial sums on those
    ghost faces back; the owner adds them to its owned entries.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import BOUNDARY, MacroMesh


@dataclass
class SlabPartition:
    rank: int
    world: int
    macro_range: tuple  # [lo, hi) global macro ids
    mesh: MacroMesh  # local mesh (local macro ids 0..hi-lo-1)
    face_global: np.ndarray  # local face -> global face id
    n_owned_faces: int
    owner_of_face: np.ndarray  # global face -> owning rank
    send_faces: dict = field(default_factory=dict)  # q -> local owned face ids (ascending global id)
    recv_faces: dict = field(default_factory=dict)  # q -> local ghost face ids owned by q (ascending global id)

    @property
    def n_local_faces(self) -> int:
        return len(self.face_global)

    @property
    def n_ghost_faces(self) -> int:
        return self.n_local_faces - self.n_owned_faces

    def dof_index(self, local_faces, Lf: int, ns: int) -> np.ndarray:
        """Flat local trace dofs of the given local faces (face-major)."""
        local_faces = np.asarray(local_faces, dtype=np.int64)
        per = Lf * ns
        return (local_faces[:, None] * per + np.arange(per)[None, :]).reshape(-1)

    def global_dofs_owned(self, Lf: int, ns: int) -> np.ndarray:
        """Global trace dof ids of this rank's owned faces, in local order."""
        per = Lf * ns
        g = self.face_global[: self.n_owned_faces]
        return (g[:, None] * per + np.arange(per)[None, :]).reshape(-1)

    def global_dofs_local(self, Lf: int, ns: int) -> np.ndarray:
        per = Lf * ns
        return (self.face_global[:, None] * per + np.arange(per)[None, :]).reshape(-1)


def slab_ranges(n_mac: int, world: int):
    cuts = [(r * n_mac) // world for r in range(world + 1)]
    return [(cuts[r], cuts[r + 1]) for r in range(world)]


def partition_mesh(mesh: MacroMesh, rank: int, world: int) -> SlabPartition:
    ranges = slab_ranges(mesh.n_macro, world)
    lo, hi = ranges[rank]
    rank_of_mac = np.empty(mesh.n_macro, dtype=np.int64)
    for r, (a, b) in enumerate(ranges):
        rank_of_mac[a:b] = r
    fm = mesh.face_macros
    owner = rank_of_mac[fm[:, 0]]
    side1_rank = np.where(fm[:, 1] >= 0, rank_of_mac[np.maximum(fm[:, 1], 0)], -1)
    local0 = owner == rank
    local1 = side1_rank == rank
    owned = np.nonzero(local0)[0]
    ghost = np.nonzero(~local0 & local1)[0]
    face_global = np.concatenate([owned, ghost])
    g2l = np.full(mesh.n_faces, -1, dtype=np.int64)
    g2l[face_global] = np.arange(len(face_global))

    nf = len(face_global)
    face_macros = np.full((nf, 2), -1, dtype=np.int64)
    face_locals = mesh.face_locals[face_global].copy()
    for side in range(2):
        glob = fm[face_global, side]
        here = (glob >= lo) & (glob < hi)
        face_macros[here, side] = glob[here] - lo
        face_locals[~here, side] = -1
    kind = mesh.face_kind[face_global].copy()
    # a face with its other side on another rank is still an interior face
    local = MacroMesh(
        vertices=mesh.vertices,
        macro_tets=mesh.macro_tets[lo:hi],
        m=mesh.m,
        face_macros=face_macros,
        face_locals=face_locals,
        face_kind=kind,
        face_label=mesh.face_label[face_global].copy(),
        corner_map=mesh.corner_map[face_global].copy(),
        periodic_offset=mesh.periodic_offset[face_global].copy(),
    )
    part = SlabPartition(rank, world, (lo, hi), local, face_global, len(owned), owner)
    # forward/reverse plans: faces with one side here and the other on rank q
    for q in range(world):
        if q == rank:
            continue
        send = owned[(side1_rank[owned] == q)]
        recv = ghost[(owner[ghost] == q)]
        if len(send):
            part.send_faces[q] = g2l[np.sort(send)]
        if len(recv):
            part.recv_faces[q] = g2l[np.sort(recv)]
    assert np.all(mesh.face_kind[face_global[part.n_owned_faces:]] != BOUNDARY)
    return part
