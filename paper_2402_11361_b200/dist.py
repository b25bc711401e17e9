"""Multi-GPU slab decomposition: halo exchanges and distributed reductions.

One process per GPU (torch.distributed, NCCL over NVLink; gloo for CPU tests).
Each rank runs the unchanged per-macro kernels on its slab (partition.py);
the only communication is what the path really needs:
  * forward halo of trace values on shared faces before every operator
    application that reads the trace (apply, residual/Jacobian, recover),
  * reverse halo of partial face sums after every operation that scatters
    onto the trace (apply, residual, rhs),
  * one exchange of the other side's face block when the block
    preconditioner is built,
  * allreduces for the Krylov dot products / norms and the Newton residual
    norm (owned trace dofs only, so every dof is counted once).

The stepper and Krylov code are unchanged: `assembly.residual/jacobian`,
`condense.condense` and `krylov.solve_trace_system` dispatch to this module
when handed a `DistDiscretization`.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .partition import partition_mesh


class Comm:
    """Thin torch.distributed wrapper; a no-op when not initialised."""

    def __init__(self):
        import torch.distributed as dist

        self.dist = dist if dist.is_available() and dist.is_initialized() else None
        self.rank = self.dist.get_rank() if self.dist else 0
        self.world = self.dist.get_world_size() if self.dist else 1
        # gloo (CPU tests, functional multi-rank checks on one GPU) moves host tensors only
        self.host_staged = bool(self.dist) and self.dist.get_backend() == "gloo"
        on_gpu = bool(self.dist) and not self.host_staged and torch.cuda.is_available()
        self.device = torch.device("cuda", torch.cuda.current_device()) if on_gpu else torch.device("cpu")

    def _wire(self, t: torch.Tensor) -> torch.Tensor:
        return t.cpu() if self.host_staged else t

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world > 1:
            w = self._wire(t)
            self.dist.all_reduce(w)
            if w is not t:
                t.copy_(w)
        return t

    def exchange(self, sends: dict, recv_counts: dict, like: torch.Tensor) -> dict:
        """Point-to-point exchange: sends[q] -> rank q, receives recv_counts[q] values from q."""
        wire_dev = torch.device("cpu") if self.host_staged else like.device
        recvs = {q: torch.empty(n, dtype=like.dtype, device=wire_dev) for q, n in recv_counts.items()}
        if self.world == 1 or (not sends and not recvs):
            return recvs
        d = self.dist
        ops = [d.P2POp(d.irecv, buf, q) for q, buf in sorted(recvs.items())]
        ops += [d.P2POp(d.isend, self._wire(t.contiguous()), q) for q, t in sorted(sends.items())]
        for req in d.batch_isend_irecv(ops):
            req.wait()
        if self.host_staged:
            recvs = {q: buf.to(like.device) for q, buf in recvs.items()}
        return recvs


def _recoverable():
    from .condense import FactorizationError
    from .krylov import PreconditionerError
    from .physics import AdmissibilityError

    return (AdmissibilityError, FactorizationError, PreconditionerError)


def collective(comm, fn):
    """Run this rank's part `fn()` and make its recoverable failure collective.

    The drivers retry a step on AdmissibilityError / FactorizationError /
    PreconditionerError (stepper.py of the reference); with slabs the failing
    macro lives on one rank, so every rank must take the same branch or the
    next halo exchange deadlocks.  One allreduce of a 3-flag vector; the rank
    that failed re-raises its own exception, the others raise the same class.
    """
    kinds = _recoverable()
    err, out = None, None
    try:
        out = fn()
    except kinds as e:
        err = e
    if comm is None or comm.world == 1:
        if err is not None:
            raise err
        return out
    flags = torch.zeros(len(kinds), dtype=torch.float64, device=comm.device)
    if err is not None:
        flags[[isinstance(err, k) for k in kinds].index(True)] = 1.0
    flags = comm.allreduce_(flags).cpu()
    if err is not None:
        raise err
    for k, v in zip(kinds, flags.tolist()):
        if v > 0:
            if k is kinds[0]:
                raise k("remote", float("nan"))
            raise k(f"{k.__name__} on another rank")
    return out


class HaloPlan:
    """Dof-level send/receive index sets of a SlabPartition."""

    def __init__(self, part, Lf: int, ns: int, device):
        per = Lf * ns
        self.per = per
        self.n_owned = part.n_owned_faces * per
        self.n_local = part.n_local_faces * per
        as_t = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int64), device=device)  # noqa: E731
        self.send = {q: as_t(part.dof_index(f, Lf, ns)) for q, f in sorted(part.send_faces.items())}
        self.recv = {q: as_t(part.dof_index(f, Lf, ns)) for q, f in sorted(part.recv_faces.items())}

    def forward(self, comm: Comm, x_owned: torch.Tensor) -> torch.Tensor:
        x_local = torch.empty(self.n_local, dtype=x_owned.dtype, device=x_owned.device)
        x_local[: self.n_owned] = x_owned
        got = comm.exchange({q: x_owned[i] for q, i in self.send.items()},
                            {q: len(i) for q, i in self.recv.items()}, x_owned)
        for q, buf in got.items():
            x_local[self.recv[q]] = buf
        return x_local

    def reverse(self, comm: Comm, y_local: torch.Tensor) -> torch.Tensor:
        y_owned = y_local[: self.n_owned].clone()
        got = comm.exchange({q: y_local[i] for q, i in self.recv.items()},
                            {q: len(i) for q, i in self.send.items()}, y_local)
        for q in sorted(got):
            y_owned.index_add_(0, self.send[q], got[q])  # unique indices per q: deterministic
        return y_owned


class DistDiscretization:
    """A rank's slab of a global macro mesh plus its halo plan.

    Presents the reference Discretization interface to the drivers with the
    trace restricted to owned faces: `n_trace` counts owned dofs, FieldState.uhat
    holds owned dofs, u and q hold the slab's macros.
    """

    is_distributed = True

    def __init__(self, global_mesh, p, params, bcs=None, source=None, quad_order=None, comm: Comm | None = None,
                 plan_device=None):
        from .discretization import Discretization

        self.comm = comm or Comm()
        self.part = partition_mesh(global_mesh, self.comm.rank, self.comm.world)
        self.local = Discretization(self.part.mesh, p, params, bcs, source, quad_order)
        for k in ("dim", "ns", "nf", "L", "Lf", "p", "params", "rm", "n_mac"):
            setattr(self, k, getattr(self.local, k))
        self.n_trace = self.part.n_owned_faces * self.Lf * self.ns
        self.global_mesh = global_mesh
        self._plan = None
        self._plan_device = plan_device

    @property
    def device(self):
        return self.local.device

    @property
    def plan(self) -> HaloPlan:
        if self._plan is None:
            dev = self._plan_device if self._plan_device is not None else self.local.device.device
            self._plan = HaloPlan(self.part, self.Lf, self.ns, dev)
        return self._plan

    # ---- host helpers -------------------------------------------------
    def local_macros(self):
        lo, hi = self.part.macro_range
        return slice(lo, hi)

    def owned_global_dofs(self):
        return self.part.global_dofs_owned(self.Lf, self.ns)

    # ---- distributed versions of the reference entry points -----------
    def forward(self, x_owned):
        return self.plan.forward(self.comm, x_owned)

    def reverse(self, y_local):
        return self.plan.reverse(self.comm, y_local)

    def _local_fields(self, fields):
        from .assembly import FieldState

        return FieldState(fields.u, fields.q, self.forward(fields.uhat))

    def residual(self, fields, ctx, frozen=None):
        from . import assembly

        lf = self._local_fields(fields)
        R_Q, R_U, R_T = collective(self.comm, lambda: assembly.residual(self.local, lf, ctx, frozen))
        return R_Q, R_U, self.reverse(R_T)

    def jacobian(self, fields, ctx):
        from . import assembly

        lf = self._local_fields(fields)
        blocks, frozen = collective(self.comm, lambda: assembly.jacobian(self.local, lf, ctx))
        blocks.dist = self
        return blocks, frozen

    def norm_sq(self, t: torch.Tensor) -> torch.Tensor:
        s = (t * t).sum().reshape(1)
        return self.comm.allreduce_(s)


class DistCondensed:
    """Condensed operator of one slab, applied with halo exchanges."""

    def __init__(self, ddisc: DistDiscretization, local_cond):
        self.dist = ddisc
        self.local = local_cond
        self.comm = ddisc.comm

    @property
    def blocks(self):
        return self.local.blocks

    def apply_trace(self, x_owned, out=None):
        y = self.dist.reverse(self.local.apply_trace(self.dist.forward(x_owned)))
        if out is not None:
            out.copy_(y)
            return out
        return y

    def rhs(self, R_Q, R_U, R_T_owned):
        zero = torch.zeros(self.dist.plan.n_local, dtype=R_U.dtype, device=R_U.device)
        return self.dist.reverse(self.local.rhs(R_Q, R_U, zero)) - R_T_owned

    def recover(self, R_Q, R_U, dtrace_owned):
        return self.local.recover(R_Q, R_U, self.dist.forward(dtrace_owned))

    def block_precond_build(self):
        return DistBlockPreconditioner(self)  # the build is collective (exchange + agreed failure)


class DistBlockPreconditioner:
    """Face-block preconditioner on owned faces; a face split across ranks gets
    the other side's block from the neighbour before factorisation."""

    def __init__(self, dcond: DistCondensed):
        from .assembly import raise_status
        from .device import current_stream

        dd = dcond.dist
        part, disc = dd.part, dd.local
        dev = disc.device
        bs = disc.Lf * disc.ns
        self.dd = dd
        self.bs = bs
        fo, so = disc.mesh.faces_of_macro, disc.mesh.sides_of_macro
        # local (macro, lf) of each local face's local side (one side per ghost face)
        mac_of = {}
        for mac in range(disc.n_mac):
            for lf in range(disc.nf):
                mac_of.setdefault(int(fo[mac, lf]), (mac, lf, int(so[mac, lf])))
        sends, recv_counts = {}, {}
        L = _lib.lib()
        for q, faces in part.recv_faces.items():  # our ghost faces owned by q: export our side
            ml = np.array([mac_of[int(f)][:2] for f in faces], dtype=np.int32)
            macs = torch.as_tensor(ml[:, 0].copy(), device=dev.device)
            lfs = torch.as_tensor(ml[:, 1].copy(), device=dev.device)
            out = torch.empty((len(faces), bs, bs), dtype=torch.float64, device=dev.device)
            _lib.check(L.mhdg_side_blocks(dev.c, dcond.blocks.c, _lib.ptr(macs), _lib.ptr(lfs), len(faces),
                                          _lib.ptr(out), current_stream()), "mhdg_side_blocks")
            sends[q] = out.reshape(-1)
        for q, faces in part.send_faces.items():
            recv_counts[q] = len(faces) * bs * bs
        like = torch.empty(1, dtype=torch.float64, device=dev.device)
        got = dd.comm.exchange(sends, recv_counts, like)
        extra = torch.zeros((part.n_local_faces, bs, bs), dtype=torch.float64, device=dev.device)
        for q, buf in got.items():
            extra[torch.as_tensor(part.send_faces[q], device=dev.device)] = buf.reshape(-1, bs, bs)
        # owned-face view of the slab's disc: ghost faces hold one side only
        self.owned_view = type(dev.c).from_buffer_copy(dev.c)
        self.owned_view.n_faces = part.n_owned_faces
        self.inverse = torch.empty((part.n_owned_faces, bs, bs), dtype=torch.float64, device=dev.device)
        status = dev.status_buffer()
        _lib.check(L.mhdg_precond_build_ext(self.owned_view, dcond.blocks.c, _lib.ptr(extra), _lib.ptr(self.inverse),
                                            _lib.ptr(status), current_stream()), "mhdg_precond_build_ext")
        collective(dd.comm, lambda: raise_status(status, "precond_build"))

    def __call__(self, v_owned):
        from .device import current_stream

        v = v_owned.contiguous()
        y = torch.empty_like(v)
        _lib.check(_lib.lib().mhdg_precond_apply(self.owned_view, _lib.ptr(self.inverse), _lib.ptr(v),
                                                 _lib.ptr(y), current_stream()), "mhdg_precond_apply")
        return y


def condense_distributed(blocks, path="schur"):
    from .condense import CondensedSchur

    return DistCondensed(blocks.dist, collective(blocks.dist.comm, lambda: CondensedSchur.build(blocks)))
