"""ORACLE (test infrastructure only): pointwise compressible-flow kernels.

CPU restatement of the reference's numpy kernel twin
(``kernels/numpy_backend.py``) for any dimension d in {2, 3}, ns = d + 2,
lambda = -2/d.  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs
may import this package; the product path never does.

  primitive_arrays   numpy_backend.py:18-27
  euler_flux         numpy_backend.py:30-39   F[pt, s, k]
  euler_jacobian     numpy_backend.py:42-63   A[pt, k, s, t] = dF[s,k]/du_t
  viscous_flux       numpy_backend.py:90-106  G[pt, s, k]
  viscous_jacobians  numpy_backend.py:109-188 dGdu[pt,k,s,t], dGdq[pt,k,l,s,t]
  stab_matrices      numpy_backend.py:191-202
  supg_tau_values    numpy_backend.py:205-212
"""

from __future__ import annotations

import numpy as np

SUPG_CD = 12.0


def _dim(u):
    return u.shape[-1] - 2


def primitive_arrays(u, gamma):
    d = _dim(u)
    rho = u[..., 0]
    v = u[..., 1 : d + 1] / rho[..., None]
    kin = 0.5 * np.einsum("...i,...i->...", v, v)
    P = (gamma - 1.0) * (u[..., d + 1] - rho * kin)
    T = gamma * P / rho
    H = (u[..., d + 1] + P) / rho
    c = np.sqrt(np.maximum(gamma * P / rho, 1e-300))
    return rho, v, P, T, H, c


def euler_flux(u, gamma):
    d = _dim(u)
    rho, v, P, _, H, _ = primitive_arrays(u, gamma)
    mom = u[:, 1 : d + 1]
    F = np.empty((u.shape[0], d + 2, d))
    F[:, 0, :] = mom
    F[:, 1 : d + 1, :] = mom[:, :, None] * v[:, None, :] + P[:, None, None] * np.eye(d)
    F[:, d + 1, :] = (rho * H)[:, None] * v
    return F


def euler_jacobian(u, gamma):
    d = _dim(u)
    E = d + 1
    rho, v, P, _, H, _ = primitive_arrays(u, gamma)
    g1 = gamma - 1.0
    kin = 0.5 * np.einsum("ni,ni->n", v, v)
    n = u.shape[0]
    A = np.zeros((n, d, d + 2, d + 2))
    I = np.eye(d)
    for k in range(d):
        A[:, k, 0, 1 + k] = 1.0
        for i in range(d):
            A[:, k, 1 + i, 0] = -v[:, i] * v[:, k] + I[i, k] * g1 * kin
            for j in range(d):
                A[:, k, 1 + i, 1 + j] = v[:, i] * I[j, k] + v[:, k] * I[i, j] - I[i, k] * g1 * v[:, j]
            A[:, k, 1 + i, E] = I[i, k] * g1
        A[:, k, E, 0] = v[:, k] * (g1 * kin - H)
        for j in range(d):
            A[:, k, E, 1 + j] = I[j, k] * H - g1 * v[:, j] * v[:, k]
        A[:, k, E, E] = gamma * v[:, k]
    return A


def _grad_parts(u, q):
    d = _dim(u)
    rho = u[:, 0]
    v = u[:, 1 : d + 1] / rho[:, None]
    gvel = (q[:, :, 1 : d + 1] - v[:, None, :] * q[:, :, 0:1]) / rho[:, None, None]
    return d, rho, v, gvel


def viscous_flux(u, q, gamma, pr, mu, re_v):
    d, rho, v, gvel = _grad_parts(u, q)
    E = d + 1
    lam = -2.0 / d
    mu_e = mu / re_v
    k_t = gamma * mu / ((gamma - 1.0) * re_v * pr)
    div = np.einsum("nll->n", gvel)
    tau = mu_e * (np.swapaxes(gvel, 1, 2) + gvel + lam * div[:, None, None] * np.eye(d))
    et = u[:, E]
    vq = np.einsum("nj,nlj->nl", v, q[:, :, 1 : d + 1])
    v2 = np.einsum("nj,nj->n", v, v)
    ge = (q[:, :, E] / rho[:, None] - et[:, None] * q[:, :, 0] / rho[:, None] ** 2
          - vq / rho[:, None] + v2[:, None] * q[:, :, 0] / rho[:, None])
    G = np.zeros((u.shape[0], d + 2, d))
    G[:, 1 : d + 1, :] = -tau
    G[:, E, :] = -np.einsum("nkj,nj->nk", tau, v) - k_t * gamma * (gamma - 1.0) * ge
    return G


def viscous_jacobians(u, q, gamma, pr, mu, re_v):
    """dG/du and dG/dq; dG/dq depends on u only."""
    d, rho, v, gvel = _grad_parts(u, q)
    E, ns = d + 1, d + 2
    n = u.shape[0]
    lam = -2.0 / d
    mu_e = mu / re_v
    kg = gamma * mu / ((gamma - 1.0) * re_v * pr) * gamma * (gamma - 1.0)
    I = np.eye(d)
    et = u[:, E]
    q0 = q[:, :, 0]
    qm = q[:, :, 1 : d + 1]

    # g[b, t] = d gvel[a, b] / d q[a, t] (same for every a)
    g = np.zeros((n, d, ns))
    for b in range(d):
        g[:, b, 1 + b] = 1.0 / rho
        g[:, b, 0] = -v[:, b] / rho
    # dtau[i, k] / dq[l, t] = mu_e (d_kl g[i,t] + d_il g[k,t] + lam d_ik g[l,t])
    dtau_q = mu_e * (np.einsum("kl,nit->niklt", I, g) + np.einsum("il,nkt->niklt", I, g)
                     + lam * np.einsum("ik,nlt->niklt", I, g))
    dGdq = np.zeros((n, d, d, ns, ns))
    dGdq[:, :, :, 1 : d + 1, :] = -np.transpose(dtau_q, (0, 2, 3, 1, 4))
    dGdq[:, :, :, E, :] = -np.einsum("nkjlt,nj->nklt", dtau_q, v)
    h = np.zeros((n, ns))
    h[:, 0] = -et / rho**2 + np.einsum("nj,nj->n", v, v) / rho
    h[:, 1 : d + 1] = -v / rho[:, None]
    h[:, E] = 1.0 / rho
    for k in range(d):
        dGdq[:, k, k, E, :] -= kg * h

    # state derivatives
    dgv = np.zeros((n, d, d, ns))  # d gvel[a, b] / d u_t
    for a in range(d):
        for b in range(d):
            dgv[:, a, b, 0] = (v[:, b] / rho * q0[:, a] - gvel[:, a, b]) / rho
            dgv[:, a, b, 1 + b] += -q0[:, a] / rho**2
    ddiv = np.einsum("nllt->nt", dgv)
    dtau_u = mu_e * (np.swapaxes(dgv, 1, 2) + dgv + lam * np.einsum("ik,nt->nikt", I, ddiv))
    tau = mu_e * (np.swapaxes(gvel, 1, 2) + gvel + lam * np.einsum("nll->n", gvel)[:, None, None] * I)
    dv = np.zeros((n, d, ns))
    for j in range(d):
        dv[:, j, 0] = -v[:, j] / rho
        dv[:, j, 1 + j] = 1.0 / rho
    v2 = np.einsum("nj,nj->n", v, v)
    vqm = np.einsum("nj,nlj->nl", v, qm)
    dge = np.zeros((n, d, ns))
    dge[:, :, 0] = (-q[:, :, E] / rho[:, None] ** 2 + 2.0 * et[:, None] * q0 / rho[:, None] ** 3
                    + 2.0 * vqm / rho[:, None] ** 2 - 3.0 * v2[:, None] * q0 / rho[:, None] ** 2)
    dge[:, :, 1 : d + 1] = (-qm / rho[:, None, None] ** 2
                            + 2.0 * v[:, None, :] * q0[:, :, None] / rho[:, None, None] ** 2)
    dge[:, :, E] = -q0 / rho[:, None] ** 2
    dGdu = np.zeros((n, d, ns, ns))
    dGdu[:, :, 1 : d + 1, :] = -np.transpose(dtau_u, (0, 2, 1, 3))
    dGdu[:, :, E, :] = (-np.einsum("nkjt,nj->nkt", dtau_u, v)
                        - np.einsum("nkj,njt->nkt", tau, dv) - kg * dge)
    return dGdu, dGdq


def stab_matrices(uhat, normals, gamma, pr, re_flow, mach):
    d = _dim(uhat)
    ns = d + 2
    _, v, _, _, _, c = primitive_arrays(uhat, gamma)
    lam = np.abs(np.einsum("ni,ni->n", v, normals)) + c
    svis = np.zeros(ns)
    svis[1 : d + 1] = 1.0
    svis[d + 1] = 1.0 / ((gamma - 1.0) * mach**2 * pr)
    S = np.zeros((uhat.shape[0], ns, ns))
    idx = np.arange(ns)
    S[:, idx, idx] = lam[:, None] + svis / re_flow
    return S, lam


def supg_tau_values(u, h, inv_dt, gamma, pr, mu, re_v):
    _, v, _, _, _, c = primitive_arrays(u, gamma)
    lam = np.linalg.norm(v, axis=-1) + c
    nu = (mu / re_v) * max(4.0 / 3.0, gamma / pr)
    return 1.0 / np.sqrt((2.0 * inv_dt) ** 2 + (2.0 * lam / h) ** 2 + (SUPG_CD * nu / h**2) ** 2)


def check_admissible(u, gamma):
    """Same test and exception as physics.py:85-94."""
    from paper_2402_11361_b200.physics import AdmissibilityError

    d = _dim(u)
    rho = u[..., 0]
    if np.any(rho <= 0.0) or not np.all(np.isfinite(rho)):
        raise AdmissibilityError("rho", float(np.min(rho)))
    kin = 0.5 * np.einsum("...i,...i->...", u[..., 1 : d + 1], u[..., 1 : d + 1]) / rho
    pres = (gamma - 1.0) * (u[..., d + 1] - kin)
    if np.any(pres <= 0.0) or not np.all(np.isfinite(pres)):
        raise AdmissibilityError("pressure", float(np.min(pres)))
