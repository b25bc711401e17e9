"""ORACLE (test infrastructure only): CPU restatement of the macro-element HDG
hot path -- assembly, second-layer condensation, matrix-free trace apply,
block preconditioner, Krylov solvers and the Newton/PTC/DIRK drivers.

Dimension-generic (d = 2, 3) numpy restatement of the reference:
  assemble_system      assembly.py:339-618  (volume 409-475, faces 477-612)
  structural applies   assembly.py:255-283, 638-724
  CondensedSchur       condense.py:54-158   (build/apply_trace/rhs/recover)
  dense_trace_operator condense.py:269-292 + assembly.py:732-865
  block_precond_build  krylov.py:194-238
  gmres / fgmres       krylov.py:51-191, solve_trace_system krylov.py:257-286
  newton/ptc/dirk      stepper.py:96-328
In 3D it is pinned against outputs of the reference itself
(tests/golden/*.npz, made by oracle/make_golden.py).  In 2D it is the
reference algebra with d generalised (ns = d+2, lambda = -2/d, d+1 faces,
face measure factor (d-1)!), plus the moving isothermal wall.

Only tests/, __graft_entry__.smoke() and bench.py (CPU baseline legs) may
import this module.  It consumes the host-side tables of a product
`Discretization` (mesh, reference tables, layouts), which are themselves
checked against the reference in tests/test_setup_vs_reference.py.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np
import scipy.linalg
from scipy.optimize import brentq

from paper_2402_11361_b200.discretization import ADIABATIC, DIRICHLET, WALL
from paper_2402_11361_b200.physics import AdmissibilityError

from . import pointwise as pw


class FactorizationError(RuntimeError):
    pass


class PreconditionerError(RuntimeError):
    pass


class NonConvergenceError(RuntimeError):
    pass


RECOVERABLE = (AdmissibilityError, FactorizationError, PreconditionerError)


# ---------------------------------------------------------------------------
# state containers
# ---------------------------------------------------------------------------


@dataclass
class Fields:
    u: np.ndarray  # (n_mac, L, ns)
    q: np.ndarray  # (n_mac, d, L, ns)
    uhat: np.ndarray  # (n_trace,)

    def copy(self):
        return Fields(self.u.copy(), self.q.copy(), self.uhat.copy())


@dataclass
class Ctx:
    dt_coeff: float = 0.0
    hist: np.ndarray | None = None
    pseudo_dt: float = np.inf
    supg_dt: float = np.inf

    @classmethod
    def steady(cls, pseudo_dt=np.inf):
        return cls(0.0, None, pseudo_dt, pseudo_dt)

    @classmethod
    def dirk_stage(cls, dt, d_row, i, stage_states, u_old):
        dii = d_row[i]
        hist = -(dii / dt) * u_old
        for j in range(i):
            hist = hist + (d_row[j] / dt) * (stage_states[j] - u_old)
        return cls(dii / dt, hist, np.inf, dt / dii)


@dataclass
class Frozen:
    supg_tau: np.ndarray
    supg_jac: np.ndarray
    face_stab: np.ndarray
    face_visc_state: np.ndarray


@dataclass
class Blocks:
    disc: object
    state_state: np.ndarray  # (M, L*ns, L*ns)
    face_state_trace: np.ndarray  # (M, nf, Lf*ns, Lf*ns)
    face_trace_state: np.ndarray
    face_trace_trace: np.ndarray
    wdgdq_vol: np.ndarray  # (M, n_sub, nq, d, d, ns, ns)
    wdgdq_face: np.ndarray  # (M, nf, n_tri*nqf, d, ns, ns)
    trace_face_scale: np.ndarray  # (M, nf)


# ---------------------------------------------------------------------------
# structural (linear, geometric) gradient-equation operators
# ---------------------------------------------------------------------------


def gather_local(disc, x):
    return x[disc.gather].reshape(disc.n_mac, disc.nf, disc.Lf, disc.ns)


def scatter_add(disc, y_loc):
    out = np.zeros(disc.n_trace)
    np.add.at(out, disc.gather.ravel(), y_loc.ravel())
    return out


def grad_mass_apply(disc, z):
    return disc.det[:, None, None, None] * np.einsum("IJ,mlJs->mlIs", disc.rm.mass, z)


def grad_mass_solve(disc, z):
    return (1.0 / disc.det)[:, None, None, None] * np.einsum("IJ,mlJs->mlIs", disc.rm.mass_inv, z)


def grad_state_apply(disc, u):
    t = np.einsum("rIJ,mJs->mrIs", disc.rm.weak_deriv, u)
    return disc.det[:, None, None, None] * np.einsum("mrl,mrIs->mlIs", disc.inv_jac, t)


def grad_trace_apply(disc, xl):
    rm = disc.rm
    out = np.zeros((disc.n_mac, disc.dim, disc.L, disc.ns))
    for lf in range(disc.nf):
        t = np.einsum("IJ,mJs->mIs", rm.face_mass, xl[:, lf])
        t = t * (disc.face_fac * disc.areas[:, lf])[:, None, None]
        out[:, :, rm.face_vol_nodes[lf], :] -= disc.normals[:, lf, :, None, None] * t[:, None]
    return out


def gradient_refresh(disc, u, uhat):
    rhs = -grad_state_apply(disc, u) - grad_trace_apply(disc, gather_local(disc, uhat))
    return grad_mass_solve(disc, rhs)


def interpolate(disc, state_fn) -> Fields:
    u, uhat = disc.nodal_interpolant(state_fn)
    return Fields(u, gradient_refresh(disc, u, uhat), uhat)


def _phys_grad(disc, K):
    return np.einsum("qar,mrl->mqal", disc.rm.grad_ref[K], disc.inv_jac)


# ---------------------------------------------------------------------------
# residual and jacobian assembly
# ---------------------------------------------------------------------------


def _kron_rows(nodes, ns):
    return (np.asarray(nodes)[:, None] * ns + np.arange(ns)[None, :]).ravel()


def _pflux(disc, u_flat, q_flat, want_jac):
    P = disc.params
    F = pw.euler_flux(u_flat, P.gamma)
    G = pw.viscous_flux(u_flat, q_flat, P.gamma, P.prandtl, P.mu, P.reynolds_acoustic)
    if not want_jac:
        return F + G, None, None
    A = pw.euler_jacobian(u_flat, P.gamma)
    dGdu, dGdq = pw.viscous_jacobians(u_flat, q_flat, P.gamma, P.prandtl, P.mu, P.reynolds_acoustic)
    return F + G, A + dGdu, dGdq


def _volume_terms(disc, fields, ctx, tder, want_jac, frozen, R_U, blocks, new_frozen):
    rm, P = disc.rm, disc.params
    M, d, ns, nq = disc.n_mac, disc.dim, disc.ns, rm.n_quad
    U, Q = fields.u, fields.q
    phi = rm.phi_vol
    inv_sdt = 0.0 if not np.isfinite(ctx.supg_dt) else 1.0 / ctx.supg_dt
    for K in range(rm.n_sub):
        conn = rm.sub_conn[K]
        gp = _phys_grad(disc, K)  # (M, nq, nloc, d)
        w = rm.w_ref[K][None, :] * disc.det[:, None]
        Uk = U[:, conn]
        u_pt = np.einsum("qa,mas->mqs", phi, Uk)
        q_pt = np.einsum("qa,mlas->mqls", phi, Q[:, :, conn])
        pw.check_admissible(u_pt, P.gamma)
        FG, Adu, dGdq = _pflux(disc, u_pt.reshape(-1, ns), q_pt.reshape(-1, d, ns), want_jac)
        R_U[:, conn] -= np.einsum("mq,mqsk,mqak->mas", w, FG.reshape(M, nq, ns, d), gp)
        if disc.source is not None:
            src = disc.source(disc.volume_quad_coords(K).reshape(-1, d)).reshape(M, nq, ns)
            R_U[:, conn] -= np.einsum("mq,qa,mqs->mas", w, phi, src)

        # SUPG with weight (A . grad w) and first-order strong residual
        gu = np.einsum("mqal,mas->mqls", gp, Uk)
        if frozen is not None:
            As = frozen.supg_jac[:, K]
            tau = frozen.supg_tau[:, K]
        else:
            As = pw.euler_jacobian(u_pt.reshape(-1, ns), P.gamma).reshape(M, nq, d, ns, ns)
            tau = pw.supg_tau_values(u_pt.reshape(-1, ns), np.repeat(disc.h_sub[:, K], nq), inv_sdt,
                                     P.gamma, P.prandtl, P.mu, P.reynolds_acoustic).reshape(M, nq)
        r_str = np.einsum("mqkut,mqkt->mqu", As, gu)
        if tder is not None:
            r_str = r_str + np.einsum("qa,mas->mqs", phi, tder[:, conn])
        W1 = np.einsum("mqkus,mqak->mqaus", As, gp)
        wt = w * tau
        R_U[:, conn] += np.einsum("mq,mqaus,mqu->mas", wt, W1, r_str)

        if want_jac:
            new_frozen.supg_tau[:, K] = tau
            new_frozen.supg_jac[:, K] = As
            blocks.wdgdq_vol[:, K] = w[:, :, None, None, None, None] * dGdq.reshape(M, nq, d, d, ns, ns)
            c = -np.einsum("mq,mqkst,mqak,qb->masbt", w, Adu.reshape(M, nq, d, ns, ns), gp, phi)
            c += np.einsum("mq,mqaus,mqbut->masbt", wt, W1, W1)
            if ctx.dt_coeff != 0.0:
                c += ctx.dt_coeff * np.einsum("mq,mqats,qb->masbt", wt, W1, phi)
            r = _kron_rows(conn, ns)
            nl = len(r)
            blocks.state_state[:, r[:, None], r[None, :]] += c.reshape(M, nl, nl)


def _face_terms(disc, fields, uh_loc, want_jac, frozen, R_U, R_T_loc, blocks, new_frozen):
    rm, P = disc.rm, disc.params
    M, d, ns, nqf = disc.n_mac, disc.dim, disc.ns, rm.n_quad_face
    E = d + 1
    U, Q = fields.u, fields.q
    pf = rm.phi_face
    I = np.eye(ns)
    for lf in range(disc.nf):
        fvn = rm.face_vol_nodes[lf]
        nvec = disc.normals[:, lf]
        is_b = disc.bc_kind[:, lf] > 0
        if want_jac:
            blocks.trace_face_scale[is_b, lf] = 0.0
        for T in range(rm.n_tri):
            tc = rm.tri_conn[T]
            sl = slice(T * nqf, (T + 1) * nqf)
            w = rm.w_face_ref[T][None, :] * (disc.face_fac * disc.areas[:, lf])[:, None]
            uh_pt = np.einsum("qa,mas->mqs", pf, uh_loc[:, lf][:, tc])
            u_pt = np.einsum("qa,mas->mqs", pf, U[:, fvn[tc]])
            q_pt = np.einsum("qa,mlas->mqls", pf, Q[:, :, fvn[tc]])
            pw.check_admissible(uh_pt, P.gamma)
            uh_f = uh_pt.reshape(-1, ns)
            q_f = q_pt.reshape(-1, d, ns)
            n_rep = np.repeat(nvec, nqf, axis=0)
            uh_v = frozen.face_visc_state[:, lf, sl].reshape(-1, ns) if frozen is not None else uh_f
            FGh = (pw.euler_flux(uh_f, P.gamma)
                   + pw.viscous_flux(uh_v, q_f, P.gamma, P.prandtl, P.mu, P.reynolds_acoustic))
            FGh = FGh.reshape(M, nqf, ns, d)
            if frozen is not None:
                S = frozen.face_stab[:, lf, sl]
            else:
                S = pw.stab_matrices(uh_f, n_rep, P.gamma, P.prandtl, P.reynolds_flow,
                                     P.mach_ref)[0].reshape(M, nqf, ns, ns)
            fn = np.einsum("mqsk,mk->mqs", FGh, nvec) + np.einsum("mqst,mqt->mqs", S, u_pt - uh_pt)
            R_U[:, fvn[tc]] += np.einsum("mq,qa,mqs->mas", w, pf, fn)
            rtr = -np.einsum("mq,qa,mqs->mas", w, pf, fn)
            if np.any(is_b):
                rtr[is_b] = 0.0
                for code, (kind, data) in disc.bc_data.items():
                    sel = disc.bc_label[:, lf] == code
                    if not np.any(sel):
                        continue
                    if kind == DIRICHLET:
                        xq = disc.face_quad_coords(lf, T)[sel]
                        bhat = uh_pt[sel] - data(xq.reshape(-1, d)).reshape(-1, nqf, ns)
                    elif kind == ADIABATIC:  # rho_hat - rho, m_hat, E_hat - E
                        bhat = uh_pt[sel].copy()
                        bhat[..., 0] -= u_pt[sel][..., 0]
                        bhat[..., E] -= u_pt[sel][..., E]
                    else:
                        e_w, u_w = data
                        uh = uh_pt[sel]
                        bhat = uh.copy()
                        bhat[..., 0] -= u_pt[sel][..., 0]
                        bhat[..., 1:E] -= uh[..., 0:1] * u_w
                        bhat[..., E] = uh[..., E] - uh[..., 0] * (e_w + 0.5 * float(u_w @ u_w))
                    rtr[sel] = np.einsum("mq,qa,mqs->mas", w[sel], pf, bhat)
            R_T_loc[:, lf][:, tc] += rtr
            if not want_jac:
                continue

            new_frozen.face_stab[:, lf, sl] = S
            new_frozen.face_visc_state[:, lf, sl] = uh_pt
            Af = pw.euler_jacobian(uh_f, P.gamma).reshape(M, nqf, d, ns, ns)
            _, dGdq = pw.viscous_jacobians(uh_v, q_f, P.gamma, P.prandtl, P.mu, P.reynolds_acoustic)
            K1 = np.einsum("mqkst,mk->mqst", Af, nvec) - S
            blocks.wdgdq_face[:, lf, sl] = np.einsum(
                "mq,mqklst,mk->mqlst", w, dGdq.reshape(M, nqf, d, d, ns, ns), nvec)
            proj = np.einsum("mq,qa,qb->mqab", w, pf, pf)
            rc = _kron_rows(tc, ns)
            nl = len(rc)
            ust = np.einsum("mqab,mqst->masbt", proj, K1).reshape(M, nl, nl)
            uss = np.einsum("mqab,mqst->masbt", proj, S).reshape(M, nl, nl)
            blocks.face_state_trace[:, lf][:, rc[:, None], rc[None, :]] += ust
            rv = _kron_rows(fvn[tc], ns)
            blocks.state_state[:, rv[:, None], rv[None, :]] += uss
            tst, ttt = -uss, -ust
            if np.any(is_b):
                tst[is_b] = 0.0
                ttt[is_b] = 0.0
                for code, (kind, data) in disc.bc_data.items():
                    sel = disc.bc_label[:, lf] == code
                    if not np.any(sel):
                        continue
                    Kuu = np.zeros((ns, ns))
                    Khh = I.copy()
                    if kind == WALL:
                        e_w, u_w = data
                        Khh[1:E, 0] = -u_w
                        Khh[E, 0] = -(e_w + 0.5 * float(u_w @ u_w))
                        Kuu[0, 0] = -1.0
                    elif kind == ADIABATIC:
                        Kuu[0, 0] = Kuu[E, E] = -1.0
                    ttt[sel] = np.einsum("mqab,st->masbt", proj[sel], Khh).reshape(-1, nl, nl)
                    tst[sel] = np.einsum("mqab,st->masbt", proj[sel], Kuu).reshape(-1, nl, nl)
            blocks.face_trace_state[:, lf][:, rc[:, None], rc[None, :]] += tst
            blocks.face_trace_trace[:, lf][:, rc[:, None], rc[None, :]] += ttt


def assemble_system(disc, fields, ctx, want_jac=True, frozen=None):
    rm = disc.rm
    M, L, Lf, ns, d, nf = disc.n_mac, disc.L, disc.Lf, disc.ns, disc.dim, disc.nf
    U = fields.u
    uh_loc = gather_local(disc, fields.uhat)
    R_U = np.zeros((M, L, ns))
    R_T_loc = np.zeros((M, nf, Lf, ns))
    R_Q = grad_mass_apply(disc, fields.q) + grad_state_apply(disc, U) + grad_trace_apply(disc, uh_loc)

    tder = None
    if ctx.dt_coeff != 0.0 or ctx.hist is not None:
        tder = ctx.dt_coeff * U
        if ctx.hist is not None:
            tder = tder + ctx.hist
        R_U += disc.det[:, None, None] * np.einsum("IJ,mJs->mIs", rm.mass, tder)

    blocks = new_frozen = None
    if want_jac:
        nqt = rm.n_tri * rm.n_quad_face
        blocks = Blocks(
            disc, np.zeros((M, L * ns, L * ns)), np.zeros((M, nf, Lf * ns, Lf * ns)),
            np.zeros((M, nf, Lf * ns, Lf * ns)), np.zeros((M, nf, Lf * ns, Lf * ns)),
            np.zeros((M, rm.n_sub, rm.n_quad, d, d, ns, ns)), np.zeros((M, nf, nqt, d, ns, ns)),
            np.ones((M, nf)))
        new_frozen = Frozen(np.zeros((M, rm.n_sub, rm.n_quad)),
                            np.zeros((M, rm.n_sub, rm.n_quad, d, ns, ns)),
                            np.zeros((M, nf, nqt, ns, ns)), np.zeros((M, nf, nqt, ns)))
        coeff = ctx.dt_coeff + (1.0 / ctx.pseudo_dt if np.isfinite(ctx.pseudo_dt) else 0.0)
        if coeff != 0.0:
            lift = np.kron(rm.mass, np.eye(ns))
            blocks.state_state += (coeff * disc.det)[:, None, None] * lift

    _volume_terms(disc, fields, ctx, tder, want_jac, frozen, R_U, blocks, new_frozen)
    _face_terms(disc, fields, uh_loc, want_jac, frozen, R_U, R_T_loc, blocks, new_frozen)
    R_T = scatter_add(disc, R_T_loc)
    if want_jac:
        return (R_Q, R_U, R_T), blocks, new_frozen
    return R_Q, R_U, R_T


def residual(disc, fields, ctx, frozen=None):
    return assemble_system(disc, fields, ctx, want_jac=False, frozen=frozen)


def jacobian(disc, fields, ctx):
    _, blocks, frozen = assemble_system(disc, fields, ctx, want_jac=True)
    return blocks, frozen


# ---------------------------------------------------------------------------
# factored block actions (assembly.py:638-724)
# ---------------------------------------------------------------------------


def state_grad_apply(blocks, z):
    disc = blocks.disc
    rm = disc.rm
    out = np.zeros((disc.n_mac, disc.L, disc.ns))
    for K in range(rm.n_sub):
        conn = rm.sub_conn[K]
        v = np.einsum("qb,mlbt->mqlt", rm.phi_vol, z[:, :, conn])
        out[:, conn] -= np.einsum("mqklst,mqlt,mqak->mas", blocks.wdgdq_vol[:, K], v, _phys_grad(disc, K))
    nqf = rm.n_quad_face
    for lf in range(disc.nf):
        fvn = rm.face_vol_nodes[lf]
        for T in range(rm.n_tri):
            tc = rm.tri_conn[T]
            v = np.einsum("qb,mlbt->mqlt", rm.phi_face, z[:, :, fvn[tc]])
            out[:, fvn[tc]] += np.einsum("mqlst,mqlt,qa->mas",
                                         blocks.wdgdq_face[:, lf, T * nqf:(T + 1) * nqf], v, rm.phi_face)
    return out


def trace_grad_apply(blocks, z):
    disc = blocks.disc
    rm = disc.rm
    nqf = rm.n_quad_face
    out = np.zeros((disc.n_mac, disc.nf, disc.Lf, disc.ns))
    for lf in range(disc.nf):
        fvn = rm.face_vol_nodes[lf]
        sc = blocks.trace_face_scale[:, lf]
        for T in range(rm.n_tri):
            tc = rm.tri_conn[T]
            v = np.einsum("qb,mlbt->mqlt", rm.phi_face, z[:, :, fvn[tc]])
            out[:, lf][:, tc] -= sc[:, None, None] * np.einsum(
                "mqlst,mqlt,qa->mas", blocks.wdgdq_face[:, lf, T * nqf:(T + 1) * nqf], v, rm.phi_face)
    return out


def state_trace_apply(blocks, xl):
    disc = blocks.disc
    M = disc.n_mac
    out = np.zeros((M, disc.L, disc.ns))
    xf = xl.reshape(M, disc.nf, -1)
    for lf in range(disc.nf):
        t = np.einsum("mab,mb->ma", blocks.face_state_trace[:, lf], xf[:, lf])
        out[:, disc.rm.face_vol_nodes[lf]] += t.reshape(M, disc.Lf, disc.ns)
    return out


def trace_state_apply(blocks, y):
    disc = blocks.disc
    M = disc.n_mac
    out = np.empty((M, disc.nf, disc.Lf, disc.ns))
    for lf in range(disc.nf):
        yf = y[:, disc.rm.face_vol_nodes[lf]].reshape(M, -1)
        out[:, lf] = np.einsum("mab,mb->ma", blocks.face_trace_state[:, lf], yf).reshape(M, disc.Lf, disc.ns)
    return out


def trace_trace_apply(blocks, xl):
    disc = blocks.disc
    M = disc.n_mac
    out = np.einsum("mfab,mfb->mfa", blocks.face_trace_trace, xl.reshape(M, disc.nf, -1))
    return out.reshape(M, disc.nf, disc.Lf, disc.ns)


# ---------------------------------------------------------------------------
# second-layer condensation (condense.py:54-158)
# ---------------------------------------------------------------------------


def schur_correction(blocks):
    """A[state,grad] A_qq^{-1} A[grad,state], dense (M, L*ns, L*ns)."""
    disc = blocks.disc
    rm = disc.rm
    M, L, ns = disc.n_mac, disc.L, disc.ns
    W = np.einsum("mrl,rIJ->mlIJ", disc.inv_jac, rm.mass_inv_weak_deriv)
    P = np.zeros((M, L, ns, L, ns))
    for K in range(rm.n_sub):
        conn = rm.sub_conn[K]
        VW = np.einsum("qb,mlbj->mqlj", rm.phi_vol, W[:, :, conn], optimize=True)
        T1 = np.einsum("mqklsr,mqak->mqlsra", blocks.wdgdq_vol[:, K], _phys_grad(disc, K), optimize=True)
        P[:, conn] -= np.einsum("mqlsra,mqlj->masjr", T1, VW, optimize=True)
    nqf = rm.n_quad_face
    for lf in range(disc.nf):
        fvn = rm.face_vol_nodes[lf]
        Wf = W[:, :, fvn]
        for T in range(rm.n_tri):
            tc = rm.tri_conn[T]
            VW = np.einsum("qb,mlbj->mqlj", rm.phi_face, Wf[:, :, tc], optimize=True)
            T1 = np.einsum("mqlsr,qa->mqlsra", blocks.wdgdq_face[:, lf, T * nqf:(T + 1) * nqf], rm.phi_face)
            P[:, fvn[tc]] += np.einsum("mqlsra,mqlj->masjr", T1, VW, optimize=True)
    return P.reshape(M, L * ns, L * ns)


def schur_matrix(blocks):
    return blocks.state_state - schur_correction(blocks)


class CondensedSchur:
    """mode "inv": explicit inverse as the reference (condense.py:67);
    mode "lu": LAPACK LU solves, the same algebra the device path uses."""

    def __init__(self, blocks, schur_inv, lu=None):
        self.blocks = blocks
        self.schur_inv = schur_inv
        self.lu = lu

    @classmethod
    def build(cls, blocks, mode="inv"):
        S = schur_matrix(blocks)
        try:
            if mode == "lu":
                return cls(blocks, None, [scipy.linalg.lu_factor(s) for s in S])
            inv = np.linalg.inv(S)
        except np.linalg.LinAlgError as exc:
            raise FactorizationError(f"singular interior Schur complement: {exc}")
        return cls(blocks, inv)

    @property
    def disc(self):
        return self.blocks.disc

    def schur_solve(self, y):
        M = self.disc.n_mac
        if self.lu is not None:
            yy = y.reshape(M, -1)
            return np.stack([scipy.linalg.lu_solve(self.lu[m], yy[m]) for m in range(M)]).reshape(y.shape)
        return np.matmul(self.schur_inv, y.reshape(M, -1, 1)).reshape(y.shape)

    def interior_elim(self, y):
        disc = self.disc
        z = grad_mass_solve(disc, grad_state_apply(disc, y))
        return trace_state_apply(self.blocks, y) - trace_grad_apply(self.blocks, z)

    def apply_trace(self, x):
        disc = self.disc
        xl = gather_local(disc, x)
        z = grad_mass_solve(disc, grad_trace_apply(disc, xl))
        y1 = -state_trace_apply(self.blocks, xl) + state_grad_apply(self.blocks, z)
        y2 = self.schur_solve(y1)
        y4 = self.interior_elim(y2) + trace_trace_apply(self.blocks, xl) - trace_grad_apply(self.blocks, z)
        return scatter_add(disc, y4)

    def apply_trace_local(self, x):
        """Unscattered local y (M, nf, Lf, ns), for kernel-level parity."""
        disc = self.disc
        xl = gather_local(disc, x)
        z = grad_mass_solve(disc, grad_trace_apply(disc, xl))
        y1 = -state_trace_apply(self.blocks, xl) + state_grad_apply(self.blocks, z)
        y2 = self.schur_solve(y1)
        return self.interior_elim(y2) + trace_trace_apply(self.blocks, xl) - trace_grad_apply(self.blocks, z)

    def rhs(self, R_Q, R_U, R_T):
        disc = self.disc
        zr = grad_mass_solve(disc, R_Q)
        t2 = self.schur_solve(R_U - state_grad_apply(self.blocks, zr))
        b_loc = self.interior_elim(t2) + trace_grad_apply(self.blocks, zr)
        return -R_T + scatter_add(disc, b_loc)

    def recover(self, R_Q, R_U, dtrace):
        disc = self.disc
        xl = gather_local(disc, dtrace)
        zr = grad_mass_solve(disc, R_Q)
        z = grad_mass_solve(disc, grad_trace_apply(disc, xl))
        y1 = -state_trace_apply(self.blocks, xl) + state_grad_apply(self.blocks, z)
        du = self.schur_solve(state_grad_apply(self.blocks, zr) - R_U + y1)
        dq = grad_mass_solve(disc, -R_Q - grad_state_apply(disc, du) - grad_trace_apply(disc, xl))
        return du, dq


def condense(blocks, path="schur", mode="inv"):
    if path != "schur":
        raise ValueError(f"unknown condensation path {path!r}")
    return CondensedSchur.build(blocks, mode)


# ---------------------------------------------------------------------------
# dense one-shot reference operator (condense.py:269-292) for small meshes
# ---------------------------------------------------------------------------


def _dense_local(blocks, mac):
    disc = blocks.disc
    rm = disc.rm
    L, Lf, ns, d, nf = disc.L, disc.Lf, disc.ns, disc.dim, disc.nf
    nq_ = L * ns
    Iq = np.eye(ns)
    # A_qq, A_qu, A_qh
    Aqq = np.kron(np.eye(d), np.kron(disc.det[mac] * rm.mass, Iq))
    Aqu = np.vstack([np.kron(disc.det[mac] * np.einsum("r,rIJ->IJ", disc.inv_jac[mac, :, l], rm.weak_deriv), Iq)
                     for l in range(d)])
    Aqh = np.zeros((d * nq_, nf * Lf * ns))
    for lf in range(nf):
        blk = np.kron(disc.face_fac * disc.areas[mac, lf] * rm.face_mass, Iq)
        ridx = _kron_rows(rm.face_vol_nodes[lf], ns)
        cidx = np.arange(lf * Lf * ns, (lf + 1) * Lf * ns)
        for l in range(d):
            Aqh[np.ix_(l * nq_ + ridx, cidx)] -= disc.normals[mac, lf, l] * blk
    # A_uq and A_hq from the stashes (materialised through the action)
    n_q = d * nq_
    Auq = np.zeros((nq_, n_q))
    Ahq = np.zeros((nf * Lf * ns, n_q))
    one = Blocks(disc, None, None, None, None, blocks.wdgdq_vol[mac:mac + 1], blocks.wdgdq_face[mac:mac + 1],
                 blocks.trace_face_scale[mac:mac + 1])

    class _Sub:
        pass

    sub = _Sub()
    for k in ("rm", "L", "Lf", "ns", "dim", "nf"):
        setattr(sub, k, getattr(disc, k))
    sub.n_mac = 1
    sub.inv_jac = disc.inv_jac[mac:mac + 1]
    one.disc = sub
    for c in range(n_q):
        e = np.zeros((1, d, L, ns))
        e.reshape(-1)[c] = 1.0
        Auq[:, c] = state_grad_apply(one, e).reshape(-1)
        Ahq[:, c] = trace_grad_apply(one, e).reshape(-1)
    Auh = np.zeros((nq_, nf * Lf * ns))
    Ahu = np.zeros((nf * Lf * ns, nq_))
    Ahh = np.zeros((nf * Lf * ns, nf * Lf * ns))
    for lf in range(nf):
        ridx = _kron_rows(rm.face_vol_nodes[lf], ns)
        cidx = np.arange(lf * Lf * ns, (lf + 1) * Lf * ns)
        Auh[np.ix_(ridx, cidx)] += blocks.face_state_trace[mac, lf]
        Ahu[np.ix_(cidx, ridx)] += blocks.face_trace_state[mac, lf]
        Ahh[np.ix_(cidx, cidx)] = blocks.face_trace_trace[mac, lf]
    A = np.block([[Aqq, Aqu], [Auq, blocks.state_state[mac]]])
    R = np.vstack([Aqh, Auh])
    C = np.hstack([Ahq, Ahu])
    return Ahh - C @ np.linalg.solve(A, R)


def dense_trace_operator(blocks):
    disc = blocks.disc
    A = np.zeros((disc.n_trace, disc.n_trace))
    for mac in range(disc.n_mac):
        idx = disc.gather[mac].ravel()
        A[np.ix_(idx, idx)] += _dense_local(blocks, mac)
    return A


# ---------------------------------------------------------------------------
# Krylov layer (krylov.py)
# ---------------------------------------------------------------------------


@dataclass
class KrylovConfig:
    restart: int = 60
    max_iter: int = 400
    abs_tol: float = 1e-12
    rel_tol: float = 1e-6
    precond: str = "block_auu_cholesky"
    inner_iter: int = 20
    inner_rel_tol: float = 0.1


@dataclass
class KrylovResult:
    x: np.ndarray
    converged: bool
    iterations: int
    residual: float
    history: list = field(default_factory=list)


def icgs(V, j, w):
    h = V[: j + 1] @ w
    w = w - V[: j + 1].T @ h
    h2 = V[: j + 1] @ w
    w = w - V[: j + 1].T @ h2
    return h + h2, w


def _givens_column(H, cs, sn, g, j):
    for i in range(j):
        t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
        H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
        H[i, j] = t
    den = np.hypot(H[j, j], H[j + 1, j])
    cs[j] = H[j, j] / den
    sn[j] = H[j + 1, j] / den
    H[j, j] = den
    g[j + 1] = -sn[j] * g[j]
    g[j] = cs[j] * g[j]


def gmres(apply_op, b, precond=None, cfg=None, x0=None):
    cfg = cfg or KrylovConfig()
    n = len(b)
    Mp = precond if precond is not None else (lambda v: v)
    x = np.zeros(n) if x0 is None else x0.copy()
    bn = np.linalg.norm(b)
    target = max(cfg.abs_tol, cfg.rel_tol * bn)
    hist = []
    if bn == 0.0:
        return KrylovResult(np.zeros(n), True, 0, 0.0, hist)
    r_true = b - apply_op(x) if x0 is not None else b.copy()
    tn = np.linalg.norm(r_true)
    if tn <= target:
        return KrylovResult(x, True, 0, tn, hist)
    total = 0
    pre_target = max(cfg.abs_tol, cfg.rel_tol * np.linalg.norm(Mp(b)))
    while total < cfg.max_iter:
        r = Mp(r_true)
        beta = np.linalg.norm(r)
        k = min(cfg.restart, cfg.max_iter - total)
        V = np.zeros((k + 1, n))
        H = np.zeros((k + 1, k))
        cs, sn, g = np.zeros(k), np.zeros(k), np.zeros(k + 1)
        g[0] = beta
        V[0] = r / beta
        jd = 0
        for j in range(k):
            w = Mp(apply_op(V[j]))
            h, w = icgs(V, j, w)
            H[: j + 1, j] = h
            hv = np.linalg.norm(w)
            H[j + 1, j] = hv
            _givens_column(H, cs, sn, g, j)
            jd = j + 1
            total += 1
            pre = abs(g[j + 1])
            hist.append((total, np.nan, pre))
            if hv <= 1e-14 * max(1.0, beta) or pre <= pre_target:
                break
            if j + 1 < k:
                V[j + 1] = w / hv
        y = scipy.linalg.solve_triangular(H[:jd, :jd], g[:jd])
        x = x + V[:jd].T @ y
        r_true = b - apply_op(x)
        tn = np.linalg.norm(r_true)
        hist[-1] = (total, tn, hist[-1][2])
        if tn <= target:
            return KrylovResult(x, True, total, tn, hist)
        pre_target = max(cfg.abs_tol, 0.1 * pre_target)
    return KrylovResult(x, False, total, tn, hist)


def fgmres(apply_op, b, inner, cfg=None, x0=None):
    cfg = cfg or KrylovConfig()
    n = len(b)
    x = np.zeros(n) if x0 is None else x0.copy()
    bn = np.linalg.norm(b)
    target = max(cfg.abs_tol, cfg.rel_tol * bn)
    hist = []
    if bn == 0.0:
        return KrylovResult(np.zeros(n), True, 0, 0.0, hist)
    r = b - apply_op(x) if x0 is not None else b.copy()
    total = 0
    while total < cfg.max_iter:
        beta = np.linalg.norm(r)
        if beta <= target:
            return KrylovResult(x, True, total, beta, hist)
        k = min(cfg.restart, cfg.max_iter - total)
        V = np.zeros((k + 1, n))
        Z = np.zeros((k, n))
        H = np.zeros((k + 1, k))
        cs, sn, g = np.zeros(k), np.zeros(k), np.zeros(k + 1)
        g[0] = beta
        V[0] = r / beta
        jd = 0
        for j in range(k):
            Z[j] = inner(V[j])
            w = apply_op(Z[j])
            h, w = icgs(V, j, w)
            H[: j + 1, j] = h
            hv = np.linalg.norm(w)
            H[j + 1, j] = hv
            _givens_column(H, cs, sn, g, j)
            jd = j + 1
            total += 1
            res = abs(g[j + 1])
            hist.append((total, res, res))
            if hv <= 1e-14 * max(1.0, beta) or res <= target:
                break
            if j + 1 < k:
                V[j + 1] = w / hv
        y = scipy.linalg.solve_triangular(H[:jd, :jd], g[:jd])
        x = x + Z[:jd].T @ y
        r = b - apply_op(x)
    return KrylovResult(x, False, total, np.linalg.norm(r), hist)


def face_trace_blocks(cond):
    """Per-face sum of both sides' trace-trace blocks in canonical order,
    symmetrised (krylov.py:201-217)."""
    blocks = cond.blocks
    disc = blocks.disc
    nf = disc.mesh.n_faces
    bs = disc.Lf * disc.ns
    B = np.zeros((nf, bs, bs))
    fo = disc.mesh.faces_of_macro
    pi = disc.gather.reshape(disc.n_mac, disc.nf, bs) - fo[:, :, None] * bs
    np.add.at(B, (fo[:, :, None, None], pi[:, :, :, None], pi[:, :, None, :]), blocks.face_trace_trace)
    return 0.5 * (B + np.swapaxes(B, -1, -2))


def block_precond_build(cond):
    B = face_trace_blocks(cond)
    nfc, bs = B.shape[0], B.shape[1]
    try:
        chol = np.linalg.cholesky(B)
    except np.linalg.LinAlgError:
        for f in range(nfc):
            try:
                np.linalg.cholesky(B[f])
            except np.linalg.LinAlgError:
                raise PreconditionerError(f"trace-trace block of face {f} is not positive definite")
        raise
    eye = np.eye(bs)
    inv = np.stack([scipy.linalg.cho_solve((chol[f], True), eye) for f in range(nfc)])

    def apply(v):
        return np.matmul(inv, v.reshape(nfc, bs, 1)).reshape(-1)

    apply.inverse = inv
    return apply


def solve_trace_system(cond, b, cfg, solver="fgmres"):
    count = {"n": 0}

    def op(v):
        count["n"] += 1
        return cond.apply_trace(v)

    pre = None if cfg.precond == "none" else block_precond_build(cond)
    if solver == "gmres":
        res = gmres(op, b, precond=pre, cfg=cfg)
    elif solver == "fgmres":
        icfg = replace(cfg, restart=max(1, cfg.inner_iter), max_iter=cfg.inner_iter,
                       rel_tol=cfg.inner_rel_tol, abs_tol=cfg.abs_tol)

        def inner(v):
            if cfg.inner_iter == 0:
                return pre(v) if pre is not None else v
            return gmres(op, v, precond=pre, cfg=icfg).x

        res = fgmres(op, b, inner, cfg=cfg)
    else:
        raise ValueError(f"unknown solver {solver!r}")
    return res, count["n"]


# ---------------------------------------------------------------------------
# nonlinear / temporal drivers (stepper.py)
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class DirkTableau:
    a: np.ndarray
    b: np.ndarray
    c: np.ndarray

    @property
    def stages(self):
        return len(self.b)

    @property
    def d(self):
        return np.linalg.inv(self.a)

    @property
    def e(self):
        return self.b @ self.d

    @classmethod
    def implicit_euler(cls):
        return cls(np.array([[1.0]]), np.array([1.0]), np.array([1.0]))

    @classmethod
    def dirk22(cls):
        g = 1.0 - np.sqrt(2.0) / 2.0
        return cls(np.array([[g, 0.0], [1.0 - g, g]]), np.array([1.0 - g, g]), np.array([g, 1.0]))

    @classmethod
    def dirk33(cls):
        al = brentq(lambda x: x**3 - 3 * x**2 + 1.5 * x - 1.0 / 6.0, 1 / 6, 1 / 2)
        c2 = (1.0 + al) / 2.0
        b1 = -(6 * al**2 - 16 * al + 1.0) / 4.0
        b2 = (6 * al**2 - 20 * al + 5.0) / 4.0
        a = np.array([[al, 0, 0], [c2 - al, al, 0], [b1, b2, al]])
        return cls(a, np.array([b1, b2, al]), np.array([al, c2, 1.0]))


@dataclass
class PtcState:
    dtau: float = 1.0
    tau_init: float = 1.0
    tau_max: float = 1e8
    prev_res: float | None = None
    printed_ratio: bool = False

    def update(self, res_u):
        if self.prev_res is not None and res_u > 0.0:
            ratio = res_u / self.prev_res if self.printed_ratio else self.prev_res / res_u
            self.dtau = min(self.dtau * ratio, self.tau_max)
        self.prev_res = res_u

    def halve(self):
        self.dtau = max(self.dtau / 2.0, 1e-12)


@dataclass
class NewtonStats:
    converged: bool = False
    iterations: int = 0
    residuals: list = field(default_factory=list)
    res_u: list = field(default_factory=list)
    dtau: list = field(default_factory=list)
    krylov_matvecs: int = 0
    krylov_iterations: int = 0
    krylov_per_step: list = field(default_factory=list)
    linear_converged: int = 0
    timings: dict = field(default_factory=lambda: {"assembly": 0.0, "condense": 0.0, "krylov": 0.0,
                                                   "recover": 0.0})


def full_norm(res):
    return float(np.sqrt(sum(float((r**2).sum()) for r in res)))


def newton_solve(disc, fields, ctx, krylov_cfg=None, solver="fgmres", abs_tol=1e-12, rel_tol=1e-6,
                 max_newton=60, ptc=None, max_retries=10, log=None, mode="inv"):
    """stepper.py:138-224.  ``mode`` picks the Schur factor representation
    ("inv": the reference's explicit inverse, condense.py:67; "lu": LAPACK LU
    solves, the algebra of the device's default packed-LU factors); ``log(st,
    fields)`` is called after every accepted step (the reference's ``log(stats)``
    hook, stepper.py:220-221, plus the accepted state for per-step goldens)."""
    cfg = krylov_cfg or KrylovConfig()
    st = NewtonStats()
    res = residual(disc, fields, ctx)
    rn = full_norm(res)
    target = max(abs_tol, rel_tol * rn)
    st.residuals.append(rn)
    st.res_u.append(float(np.linalg.norm(res[1])))
    if ptc is not None:
        ptc.prev_res = st.res_u[-1]
    for it in range(max_newton):
        if rn <= target:
            st.converged = True
            break
        retries = 0
        while True:
            cur = ctx
            if ptc is not None:
                cur = Ctx(ctx.dt_coeff, ctx.hist, ptc.dtau, ptc.dtau)
                st.dtau.append(ptc.dtau)
            try:
                t0 = time.perf_counter()
                blocks, _ = jacobian(disc, fields, cur)
                t1 = time.perf_counter()
                cond = condense(blocks, mode=mode)
                t2 = time.perf_counter()
                b = cond.rhs(*res)
                lin, nmv = solve_trace_system(cond, b, cfg, solver)
                t3 = time.perf_counter()
                du, dq = cond.recover(res[0], res[1], lin.x)
                t4 = time.perf_counter()
                for k, dt_ in zip(("assembly", "condense", "krylov", "recover"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
                    st.timings[k] += dt_
                st.krylov_matvecs += nmv
                st.krylov_iterations += lin.iterations
                st.linear_converged += int(lin.converged)
                trial = Fields(fields.u + du, fields.q + dq, fields.uhat + lin.x)
                new_res = residual(disc, trial, ctx)
                new_norm = full_norm(new_res)
                if not np.isfinite(new_norm) or new_norm > 100.0 * max(rn, abs_tol):
                    raise AdmissibilityError("residual growth", new_norm)
                break
            except RECOVERABLE:
                retries += 1
                if ptc is None or retries > max_retries:
                    raise
                ptc.halve()
        fields.u, fields.q, fields.uhat = trial.u, trial.q, trial.uhat
        res, rn = new_res, new_norm
        st.iterations = it + 1
        st.residuals.append(rn)
        st.res_u.append(float(np.linalg.norm(res[1])))
        if ptc is not None:
            ptc.update(st.res_u[-1])
        st.krylov_per_step.append(st.krylov_iterations - sum(st.krylov_per_step))
        if log is not None:
            log(st, fields)
    else:
        st.converged = rn <= target
    return st


def ptc_steady_solve(disc, fields, krylov_cfg=None, solver="fgmres", abs_tol=1e-10, rel_tol=1e-8,
                     max_newton=120, tau_init=1.0, tau_max=1e8, ser_printed_ratio=False, log=None, mode="inv"):
    """stepper.py:227-262 (``mode``/``log`` as in newton_solve)."""
    ptc = PtcState(dtau=tau_init, tau_init=tau_init, tau_max=tau_max, printed_ratio=ser_printed_ratio)
    st = newton_solve(disc, fields, Ctx.steady(), krylov_cfg=krylov_cfg, solver=solver, abs_tol=abs_tol,
                      rel_tol=rel_tol, max_newton=max_newton, ptc=ptc, log=log, mode=mode)
    if not st.converged:
        raise NonConvergenceError(f"steady solve stalled at {st.residuals[-1]:.3e}")
    return st, ptc


def dirk_advance(disc, fields, dt, tableau, krylov_cfg=None, solver="fgmres", abs_tol=1e-12, rel_tol=1e-8,
                 max_newton=30, max_dt_retries=4, mode="inv"):
    """stepper.py:265-328 (``mode`` as in newton_solve)."""
    if abs(tableau.c[-1] - 1.0) > 1e-12:
        raise NotImplementedError("tableaus with c_s != 1 require a trailing trace/gradient solve")
    d, e = tableau.d, tableau.e
    u_old = fields.u.copy()
    start = fields.copy()
    dt_cur = float(dt)
    for attempt in range(max_dt_retries + 1):
        try:
            all_st, stages = [], []
            for i in range(tableau.stages):
                ctx = Ctx.dirk_stage(dt_cur, d[i], i, stages, u_old)
                st = newton_solve(disc, fields, ctx, krylov_cfg=krylov_cfg, solver=solver, abs_tol=abs_tol,
                                  rel_tol=rel_tol, max_newton=max_newton, mode=mode)
                if not st.converged:
                    raise NonConvergenceError(f"stage {i} did not converge")
                all_st.append(st)
                stages.append(fields.u.copy())
            break
        except (NonConvergenceError, *RECOVERABLE):
            if attempt == max_dt_retries:
                raise
            dt_cur *= 0.5
            fields.u[:] = start.u
            fields.q[:] = start.q
            fields.uhat[:] = start.uhat
    u_new = (1.0 - e.sum()) * u_old
    for j in range(tableau.stages):
        u_new += e[j] * stages[j]
    fields.u[:] = u_new
    return all_st, dt_cur
