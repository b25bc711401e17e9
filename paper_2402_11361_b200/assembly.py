"""Residuals and Jacobian blocks on the device (the reference's assembly API).

Mirrors assembly.py of the reference: FieldState (assembly.py:37-51),
StageContext (assembly.py:54-81), FrozenCoeffs (assembly.py:84-96),
LocalBlocks (assembly.py:293-320), residual() (assembly.py:621-623) and
jacobian() (assembly.py:626-629).  Arrays are torch CUDA float64 tensors in
the reference layouts; the work is done by the sm_100a kernels behind
mhdg_assemble (paper_2402_11361_b200/csrc/assemble.cu).
"""

from __future__ import annotations

import math
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .device import current_stream
from .discretization import ConfigError, Discretization  # noqa: F401  (re-export)
from .physics import AdmissibilityError

NS3 = 5


@dataclass
class FieldState:
    u: torch.Tensor  # (n_mac, L, ns)
    q: torch.Tensor  # (n_mac, d, L, ns)
    uhat: torch.Tensor  # (n_trace,)

    def copy(self) -> "FieldState":
        return FieldState(self.u.clone(), self.q.clone(), self.uhat.clone())

    def axpy(self, alpha, du, dq, duhat) -> None:
        self.u += alpha * du
        self.q += alpha * dq
        self.uhat += alpha * duhat


@dataclass
class StageContext:
    dt_coeff: float = 0.0
    hist: torch.Tensor | None = None
    pseudo_dt: float = math.inf
    supg_dt: float = math.inf

    @classmethod
    def steady(cls, pseudo_dt: float = math.inf) -> "StageContext":
        return cls(0.0, None, pseudo_dt, pseudo_dt)

    @classmethod
    def dirk_stage(cls, dt, d_row, stage_idx, stage_states, u_old) -> "StageContext":
        d_ii = float(d_row[stage_idx])
        hist = -(d_ii / dt) * u_old
        for j in range(stage_idx):
            hist = hist + (float(d_row[j]) / dt) * (stage_states[j] - u_old)
        return cls(d_ii / dt, hist, math.inf, dt / d_ii)


@dataclass
class FrozenCoeffs:
    supg_tau: torch.Tensor
    supg_jac: torch.Tensor
    face_stab: torch.Tensor
    face_visc_state: torch.Tensor

    def c_struct(self):
        c = _lib.Frozen()
        c.supg_tau, c.supg_jac = _lib.ptr(self.supg_tau), _lib.ptr(self.supg_jac)
        c.face_stab, c.face_visc_state = _lib.ptr(self.face_stab), _lib.ptr(self.face_visc_state)
        return c

    @classmethod
    def empty(cls, disc, n_mac: int | None = None):
        rm, M, d, ns, nf = disc.rm, disc.n_mac if n_mac is None else n_mac, disc.dim, disc.ns, disc.nf
        dev = disc.device.device
        nqt = rm.n_tri * rm.n_quad_face
        z = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
        return cls(z(M, rm.n_sub, rm.n_quad), z(M, rm.n_sub, rm.n_quad, d, ns, ns), z(M, nf, nqt, ns, ns),
                   z(M, nf, nqt, ns))


class LocalBlocks:
    """Per-macro Jacobian data in the reference's factored/stashed form."""

    KEYS = ("state_state", "face_state_trace", "face_trace_state", "face_trace_trace", "wdgdq_vol",
            "wdgdq_face", "trace_face_scale")

    def __init__(self, disc, **arrays):
        self.disc = disc
        for k in self.KEYS:
            setattr(self, k, arrays[k])
        self._c = None

    @classmethod
    def empty(cls, disc, n_mac: int | None = None, with_state_state: bool = True):
        """Uninitialised blocks for every macro, or (coupling-recompute windows) for `n_mac`
        macros, optionally without state_state (a NULL pointer in the C struct)."""
        rm, M, d, ns, nf, L, Lf = disc.rm, disc.n_mac if n_mac is None else n_mac, disc.dim, disc.ns, disc.nf, disc.L, disc.Lf
        dev = disc.device.device
        z = lambda *s: torch.empty(s, dtype=torch.float64, device=dev)  # noqa: E731
        return cls(disc, state_state=z(M, L * ns, L * ns) if with_state_state else None, face_state_trace=z(M, nf, Lf * ns, Lf * ns),
                   face_trace_state=z(M, nf, Lf * ns, Lf * ns), face_trace_trace=z(M, nf, Lf * ns, Lf * ns),
                   wdgdq_vol=z(M, rm.n_sub, rm.n_quad, d, d, ns, ns),
                   wdgdq_face=z(M, nf, rm.n_tri * rm.n_quad_face, d, ns, ns), trace_face_scale=z(M, nf))

    @classmethod
    def from_arrays(cls, disc, arrays: dict):
        """Upload host arrays (e.g. the oracle's blocks) in the reference layout."""
        dev = disc.device.device
        return cls(disc, **{k: torch.as_tensor(np.ascontiguousarray(arrays[k]), dtype=torch.float64, device=dev)
                            for k in cls.KEYS})

    @property
    def c(self):
        if self._c is None:
            c = _lib.Blocks()
            for k in self.KEYS:
                t = getattr(self, k)
                assert t is None or (t.is_contiguous() and t.dtype == torch.float64)
                setattr(c, k, _lib.ptr(t))
            self._c = c
        return self._c

    @property
    def n_state(self) -> int:
        return self.disc.L * self.disc.ns

    @property
    def n_grad(self) -> int:
        return self.disc.dim * self.disc.L * self.disc.ns

    def to_host(self) -> dict:
        return {k: getattr(self, k).cpu().numpy() for k in self.KEYS}


# MHDG_APPLY_REPR=recompute (or jacobian(..., recompute=True)): jacobian() returns the
# linearisation point instead of assembled blocks (the coupling-recompute representation)
# macros per window (MHDG_RECOMPUTE_CHUNK, read when the blocks are created)
RECOMPUTE_CHUNK = 4096


class RecomputeBlocks:
    """The linearisation point (u, q, uhat, stage context) standing in for LocalBlocks under
    the coupling-recompute representation (B_min; "store
    only S^-1 and transformation data"): condense() factors S window by window from it and
    the condensed operator re-forms the coupling blocks of a window of `chunk` macros
    before each local apply (condense.CondensedRecompute).  Per macro it keeps (1 + d) L ns
    doubles instead of the blocks' (L ns)^2 + 3 nf (Lf ns)^2 + stashes."""

    def __init__(self, disc, fields: FieldState, ctx: StageContext, chunk: int | None = None):
        self.disc = disc
        cp = lambda t: t.detach().clone(memory_format=torch.contiguous_format)  # noqa: E731
        self.u, self.q, self.uhat = cp(fields.u), cp(fields.q), cp(fields.uhat)
        self.ctx = ctx
        chunk = chunk or int(os.environ.get("MHDG_RECOMPUTE_CHUNK", RECOMPUTE_CHUNK))
        self.chunk = max(1, min(int(chunk), disc.n_mac))
        self.stage, self._hist_keep = _stage_struct(ctx, disc)
        self.flow = _flow_struct(disc.params)

    def assemble_window(self, mac0: int, count: int, want_jac: int, window: LocalBlocks, status,
                        frozen: FrozenCoeffs | None = None, res=(None, None, None)) -> None:
        """mhdg_assemble_window for macros [mac0, mac0 + count): want_jac = 1 blocks + frozen
        coefficients + residual vectors (all window-sized), 2 the couplings only."""
        rc = _lib.lib().mhdg_assemble_window(
            self.disc.device.c, self.flow, self.stage, _lib.ptr(self.u), _lib.ptr(self.q), _lib.ptr(self.uhat),
            _lib.ptr(res[0]), _lib.ptr(res[1]), _lib.ptr(res[2]), int(want_jac), window.c,
            frozen.c_struct() if frozen is not None else None, int(mac0), int(count), _lib.ptr(status),
            current_stream())
        _lib.check(rc, "mhdg_assemble_window")


def raise_status(status: torch.Tensor, what: str) -> None:
    """Map the device status word to the reference's exception classes."""
    st = status.cpu().numpy()
    code = int(st[0])
    if code == _lib.MHDG_OK:
        return
    val = float(np.array([st[3]], dtype=np.int32).view(np.float32)[0])
    if code == _lib.MHDG_ERR_ADMISSIBILITY:
        raise AdmissibilityError("rho" if st[2] == 0 else "pressure", val)
    if code == _lib.MHDG_ERR_FACTORIZATION:
        from .condense import FactorizationError

        raise FactorizationError(f"singular interior Schur complement (macro {int(st[1])})")
    if code == _lib.MHDG_ERR_PRECONDITIONER:
        from .krylov import PreconditionerError

        raise PreconditionerError(f"trace-trace block of face {int(st[1])} is not positive definite")
    raise RuntimeError(f"{what}: device status {st.tolist()}")


def _flow_struct(params):
    f = _lib.Flow()
    f.gamma, f.prandtl, f.re_acoustic = params.gamma, params.prandtl, params.reynolds_acoustic
    f.mach_ref, f.mu, f.re_flow = params.mach_ref, params.mu, params.reynolds_flow
    return f


def _stage_struct(ctx, disc):
    s = _lib.Stage()
    s.dt_coeff = float(ctx.dt_coeff)
    hist = ctx.hist
    if hist is not None:
        if not isinstance(hist, torch.Tensor):
            hist = torch.as_tensor(np.asarray(hist), dtype=torch.float64, device=disc.device.device)
        hist = hist.contiguous()
    s.hist = _lib.ptr(hist)
    s.pseudo_dt = float(ctx.pseudo_dt)
    s.supg_dt = float(ctx.supg_dt)
    return s, hist


def assemble_system(disc, fields: FieldState, ctx: StageContext, want_jac: bool = True,
                    frozen: FrozenCoeffs | None = None):
    """Residuals (R_Q, R_U, R_trace) and optionally blocks + frozen coefficients
    (assembly.py:339-618).  Raises AdmissibilityError like the reference."""
    dd = disc.device
    dev = dd.device
    M, d, L, ns = disc.n_mac, disc.dim, disc.L, disc.ns
    R_Q = torch.empty((M, d, L, ns), dtype=torch.float64, device=dev)
    R_U = torch.empty((M, L, ns), dtype=torch.float64, device=dev)
    R_Tl = torch.empty(dd.n_local_trace, dtype=torch.float64, device=dev)
    R_T = torch.empty(disc.n_trace, dtype=torch.float64, device=dev)
    blocks = LocalBlocks.empty(disc) if want_jac else None
    new_frozen = FrozenCoeffs.empty(disc) if want_jac else None
    status = dd.status_buffer()
    stage, hist_keep = _stage_struct(ctx, disc)
    flow = _flow_struct(disc.params)
    fo = new_frozen.c_struct() if want_jac else None
    fi = frozen.c_struct() if frozen is not None else None
    u_c = _lib.arg(fields.u, M * L * ns, "fields.u")  # bound locals: alive across the call
    q_c = _lib.arg(fields.q, M * d * L * ns, "fields.q")
    uh_c = _lib.arg(fields.uhat, disc.n_trace, "fields.uhat")
    rc = _lib.lib().mhdg_assemble(
        dd.c, flow, stage, _lib.ptr(u_c), _lib.ptr(q_c),
        _lib.ptr(uh_c), _lib.ptr(R_Q), _lib.ptr(R_U), _lib.ptr(R_Tl), _lib.ptr(R_T),
        int(want_jac), blocks.c if want_jac else None, fo, fi, _lib.ptr(status), current_stream())
    _lib.check(rc, "mhdg_assemble")
    raise_status(status, "assemble")
    del hist_keep
    if want_jac:
        return (R_Q, R_U, R_T), blocks, new_frozen
    return R_Q, R_U, R_T


def residual(disc, fields, ctx, frozen: FrozenCoeffs | None = None):
    if getattr(disc, "is_distributed", False):
        return disc.residual(fields, ctx, frozen)
    return assemble_system(disc, fields, ctx, want_jac=False, frozen=frozen)


def jacobian(disc, fields, ctx, recompute: bool | None = None):
    """Blocks + frozen coefficients (assembly.py:626-629).  With `recompute` (default:
    MHDG_APPLY_REPR=recompute) the blocks are a RecomputeBlocks -- nothing is assembled
    here, condense() and the condensed operator form windows of blocks on demand -- and
    no frozen coefficients are returned."""
    if getattr(disc, "is_distributed", False):
        return disc.jacobian(fields, ctx)
    if recompute is None:
        recompute = os.environ.get("MHDG_APPLY_REPR", "matrix_free") == "recompute"
    if recompute:
        return RecomputeBlocks(disc, fields, ctx), None
    _, blocks, frozen = assemble_system(disc, fields, ctx, want_jac=True)
    return blocks, frozen


def gradient_refresh(disc, u: torch.Tensor, uhat: torch.Tensor) -> torch.Tensor:
    """q = A_qq^-1 (-A_qu u - A_qh uhat) on the device (assembly.py:247-252)."""
    dd = disc.device
    q = torch.empty((disc.n_mac, disc.dim, disc.L, disc.ns), dtype=torch.float64, device=dd.device)
    u_c = _lib.arg(u, disc.n_mac * disc.L * disc.ns, "u")
    uh_c = _lib.arg(uhat, disc.n_trace, "uhat")
    rc = _lib.lib().mhdg_gradient_refresh(dd.c, _lib.ptr(u_c), _lib.ptr(uh_c), _lib.ptr(q), current_stream())
    _lib.check(rc, "mhdg_gradient_refresh")
    return q


def to_device_fields(disc, u, q, uhat) -> FieldState:
    dev = disc.device.device
    t = lambda a: torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device=dev)  # noqa: E731
    return FieldState(t(u), t(q), t(uhat))


def interpolate(disc, state_fn) -> FieldState:
    """Nodal + owner-side trace interpolation, gradient refreshed on the device
    (Discretization.interpolate, assembly.py:228-245)."""
    if getattr(disc, "is_distributed", False):
        u, uhat = disc.local.nodal_interpolant(state_fn)
        dev = disc.device.device
        ut = torch.as_tensor(u, dtype=torch.float64, device=dev)
        uh = torch.as_tensor(uhat[: disc.n_trace], dtype=torch.float64, device=dev)
        return FieldState(ut, gradient_refresh(disc.local, ut, disc.forward(uh)), uh)
    u, uhat = disc.nodal_interpolant(state_fn)
    dev = disc.device.device
    ut = torch.as_tensor(u, dtype=torch.float64, device=dev)
    uh = torch.as_tensor(uhat, dtype=torch.float64, device=dev)
    return FieldState(ut, gradient_refresh(disc, ut, uh), uh)


def zero_fields(disc) -> FieldState:
    dev = disc.device.device
    return FieldState(torch.zeros((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device=dev),
                      torch.zeros((disc.n_mac, disc.dim, disc.L, disc.ns), dtype=torch.float64, device=dev),
                      torch.zeros(disc.n_trace, dtype=torch.float64, device=dev))
