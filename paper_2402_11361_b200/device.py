"""Device-resident discretization tables (torch tensors) and their C struct.

Built once per Discretization.  Everything the kernels read per launch lives
here: reference tables (plus three derived, macro-independent tables: Gf =
M^-1[:, fvn[f]] Mf, PM = phi M^-1 D per volume quadrature point and PMf per
face quadrature point), per-macro geometry, the int32 trace gather and its
inverse (two sorted local sources per trace dof), inverse-incidence CSR
tables that make every accumulation deterministic, and boundary data.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib


def _csr(n_rows: int, keys: np.ndarray, vals: np.ndarray):
    """CSR of vals grouped by keys (stable: original order inside a row)."""
    order = np.argsort(keys, kind="stable")
    counts = np.bincount(keys, minlength=n_rows)
    ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    return ptr, vals[order].astype(np.int32)


def cuda_device():
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the macro-element HDG path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def current_stream():
    return torch.cuda.current_stream().cuda_stream


class DeviceDisc:
    def __init__(self, disc):
        self.disc = disc
        dev = self.device = cuda_device()
        rm, d = disc.rm, disc.dim
        f64 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=dev)  # noqa: E731
        i32 = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32), device=dev)  # noqa: E731
        t = {}
        fvn = rm.face_vol_nodes
        t["mass"] = f64(rm.mass)
        t["mass_inv"] = f64(rm.mass_inv)
        # tables streamed by bulk copies are padded so an even-rounded piece
        # never reads past the allocation
        pad2 = lambda a: np.concatenate([np.ascontiguousarray(a, dtype=np.float64).ravel(), np.zeros(2)])  # noqa: E731
        t["minv_d"] = f64(pad2(rm.mass_inv_weak_deriv))
        t["weak_deriv"] = f64(rm.weak_deriv)
        t["gf"] = f64(pad2(np.stack([rm.mass_inv[:, fvn[f]] @ rm.face_mass for f in range(disc.nf)])))
        t["face_mass"] = f64(rm.face_mass)
        t["face_vol_nodes"] = i32(fvn)
        t["sub_conn"] = i32(rm.sub_conn)
        t["phi_vol"] = f64(rm.phi_vol)
        t["grad_ref"] = f64(rm.grad_ref)
        t["w_ref"] = f64(rm.w_ref)
        t["tri_conn"] = i32(rm.tri_conn)
        t["phi_face"] = f64(rm.phi_face)
        t["w_face_ref"] = f64(rm.w_face_ref)
        MD = rm.mass_inv_weak_deriv  # (d, L, L)
        t["pm_vol"] = f64(np.einsum("qb,rKbj->Kqrj", rm.phi_vol, MD[:, rm.sub_conn, :]))
        pmf = np.empty((disc.nf, rm.n_tri, rm.n_quad_face, d, disc.L))
        for f in range(disc.nf):
            pmf[f] = np.einsum("qb,rTbj->Tqrj", rm.phi_face, MD[:, fvn[f][rm.tri_conn], :])
        t["pm_face"] = f64(pmf)
        L, Lf = disc.L, disc.Lf
        ptr, ent = _csr(L, rm.sub_conn.ravel(), np.arange(rm.sub_conn.size))
        t["vn_ptr"], t["vn_sub"] = i32(ptr), i32(ent)
        ptr, ent = _csr(L, fvn.ravel(), np.arange(fvn.size))
        t["vf_ptr"], t["vf_ent"] = i32(ptr), i32(ent)
        ptr, ent = _csr(Lf, rm.tri_conn.ravel(), np.arange(rm.tri_conn.size))
        t["fn_ptr"], t["fn_ent"] = i32(ptr), i32(ent)
        t["det"] = f64(disc.det)
        t["inv_jac"] = f64(disc.inv_jac)
        t["normals"] = f64(disc.normals)
        t["areas"] = f64(disc.areas)
        t["h_sub"] = f64(disc.h_sub)
        if disc.n_mac * disc.nf * Lf * disc.ns >= 2**31:
            raise ValueError("local trace index space exceeds int32")
        t["gather"] = i32(disc.gather)
        t["scatter_src"] = i32(disc.scatter_sources())
        wall_e, wall_u, u_dir = disc.boundary_tables()
        t["bc_kind"] = i32(disc.bc_kind)
        t["wall_e"] = f64(wall_e)
        t["wall_u"] = f64(wall_u)
        t["u_dir"] = f64(u_dir)
        src = disc.source_table()
        t["source"] = f64(src) if src is not None else None
        t["face_macros"] = i32(disc.mesh.face_macros)
        t["face_locals"] = i32(disc.mesh.face_locals)
        fnodes = np.unique(fvn)
        n2f = np.full(L, -1, dtype=np.int64)
        n2f[fnodes] = np.arange(len(fnodes))
        t["node_to_face"] = i32(n2f)
        t["minv_d_face"] = f64(pad2(rm.mass_inv_weak_deriv[:, fnodes, :]))
        self.n_face_nodes = len(fnodes)
        # distinct per-sub-element gradient tables (exact comparison)
        G = np.ascontiguousarray(rm.grad_ref).reshape(rm.n_sub, -1)
        cls, cls_of = np.unique(G, axis=0, return_inverse=True)
        t["grad_cls"] = f64(cls)
        t["grad_cls_of"] = i32(cls_of.ravel())
        self.n_grad_cls = len(cls)
        self.t = t

        c = _lib.Disc()
        c.dim, c.ns, c.nf = d, disc.ns, disc.nf
        c.n_mac, c.n_faces, c.n_trace = disc.n_mac, disc.mesh.n_faces, disc.n_trace
        c.L, c.Lf = L, Lf
        c.n_sub, c.nloc, c.nq = rm.n_sub, rm.n_loc, rm.n_quad
        c.n_tri, c.nlocf, c.nqf = rm.n_tri, rm.n_loc_face, rm.n_quad_face
        c.face_fac = disc.face_fac
        c.n_face_nodes = self.n_face_nodes
        c.n_grad_cls = self.n_grad_cls
        for name, tensor in t.items():
            setattr(c, name, _lib.ptr(tensor))
        self.c = c

    # ------------------------------------------------------------------
    @property
    def n_local_trace(self) -> int:
        d = self.disc
        return d.n_mac * d.nf * d.Lf * d.ns

    def status_buffer(self):
        return torch.zeros(4, dtype=torch.int32, device=self.device)
