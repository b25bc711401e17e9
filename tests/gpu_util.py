"""Helpers shared by the GPU parity tests."""

import numpy as np
import pytest
import torch

import oracle.hdg_oracle as O
from paper_2402_11361_b200.assembly import LocalBlocks


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def upload_blocks(disc, ob):
    return LocalBlocks.from_arrays(disc, {k: getattr(ob, k) for k in LocalBlocks.KEYS})


def perturbed_fields(disc, state_fn, seed, amp_u=1e-3, amp_q=1e-2):
    f = O.interpolate(disc, state_fn)
    rng = np.random.default_rng(seed)
    f.u = f.u + amp_u * rng.standard_normal(f.u.shape) * np.abs(f.u).max()
    f.uhat = f.uhat + amp_u * rng.standard_normal(f.uhat.shape) * np.abs(f.uhat).max()
    f.q = f.q + amp_q * rng.standard_normal(f.q.shape)
    return f


def subset_disc(disc, idx):
    """A host Discretization restricted to the macros `idx` (sorted), sharing the
    global trace numbering: the oracle run on it reproduces exactly those macros'
    local operators (every per-macro array is sliced; gather still indexes the
    full trace vector, so a global x gathers the same local traces)."""
    import copy

    sub = copy.copy(disc)
    idx = np.asarray(idx)
    sub.n_mac = len(idx)
    for k in ("det", "inv_jac", "jac", "origin", "normals", "areas", "h_sub", "gather", "bc_kind", "bc_label"):
        setattr(sub, k, getattr(disc, k)[idx])
    sub._device = None
    return sub


class _SubMesh:
    """The few mesh attributes the device tables read (device.DeviceDisc)."""

    def __init__(self, n_faces, face_macros, face_locals, m):
        self.n_faces, self.face_macros, self.face_locals, self.m = n_faces, face_macros, face_locals, m


def compact_subset_disc(disc, idx):
    """A Discretization of only the macros `idx` with its own compact trace numbering:
    the faces they touch, renumbered 0..F'-1 in ascending global id (the per-face dof
    layout (f Lf + g) ns + s is kept), so device tables (scatter sources, face lists)
    can be built for the subset.  Returns (sub_disc, global_dofs) with global_dofs[i]
    the global trace dof of compact dof i."""
    import copy

    idx = np.asarray(idx)
    sub = subset_disc(disc, idx)
    per = disc.Lf * disc.ns
    fo = disc.mesh.faces_of_macro[idx]
    faces = np.unique(fo)
    new_of = np.full(disc.mesh.n_faces, -1, dtype=np.int64)
    new_of[faces] = np.arange(len(faces))
    g = disc.gather[idx]
    sub.gather = new_of[g // per] * per + g % per
    sub.n_trace = len(faces) * per
    pos = np.full(disc.n_mac, -1, dtype=np.int64)
    pos[idx] = np.arange(len(idx))
    fm = disc.mesh.face_macros[faces]
    fmap = np.where(fm >= 0, pos[np.maximum(fm, 0)], -1)
    fl = np.where(fmap >= 0, disc.mesh.face_locals[faces], -1)
    # side 0 must be present for the preconditioner's face loop: swap sides where only side 1 is
    swap = (fmap[:, 0] < 0) & (fmap[:, 1] >= 0)
    fmap[swap] = fmap[swap][:, ::-1]
    fl[swap] = fl[swap][:, ::-1]
    sub.mesh = _SubMesh(len(faces), fmap, fl, disc.mesh.m)
    sub._device = None
    glob = (faces[:, None] * per + np.arange(per)[None, :]).reshape(-1)
    return sub, glob
