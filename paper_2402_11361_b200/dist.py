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

    def exchange_start(self, sends: dict, recv_bufs: dict):
        """Post the sends and receives (into the given contiguous views) and return a
        wait() that makes the current stream wait for them: with NCCL the transfers run
        on the communicator's stream while the caller keeps launching kernels."""
        if self.world == 1 or (not sends and not recv_bufs):
            return lambda: None
        if self.host_staged:
            like = next(iter(recv_bufs.values()), None)  # a rank may only send (it owns every shared face)
            if like is None:
                like = next(iter(sends.values()))
            got = self.exchange(sends, {q: b.numel() for q, b in recv_bufs.items()}, like)
            for q, b in recv_bufs.items():
                b.copy_(got[q])
            return lambda: None
        d = self.dist
        ops = [d.P2POp(d.irecv, buf, q) for q, buf in sorted(recv_bufs.items())]
        ops += [d.P2POp(d.isend, t, q) for q, t in sorted(sends.items())]
        reqs = d.batch_isend_irecv(ops)

        def wait():
            for r in reqs:
                r.wait()

        return wait

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


def _start_exchange(comm, sends: dict, recv_bufs: dict):
    """Start a point-to-point exchange into preallocated receive views; returns a
    wait() that makes the current stream wait for the received data (NCCL) or
    nothing (synchronous communicators)."""
    if hasattr(comm, "exchange_start"):
        return comm.exchange_start(sends, recv_bufs)
    like = next(iter(recv_bufs.values()), next(iter(sends.values()), None))
    got = comm.exchange(sends, {q: b.numel() for q, b in recv_bufs.items()}, like)
    for q, b in recv_bufs.items():
        b.copy_(got[q])
    return lambda: None


def _segments(buf: torch.Tensor, counts: dict) -> dict:
    out, o = {}, 0
    for q in sorted(counts):
        out[q] = buf[o: o + counts[q]]
        o += counts[q]
    return out


class HaloPlan:
    """Dof-level send/receive index sets of a SlabPartition, as int32 device tables
    for the library's halo kernels (mhdg_halo_gather / _scatter / _face_reduce_remote).

    Per neighbour q (ascending), faces in ascending global id on both sides:
      fwd_send -- owned dofs q holds as ghosts (x sent forward; y received back),
      fwd_recv -- this rank's ghost dofs owned by q (x received; y sent back),
      rev_send -- the local flat y_loc entries of those ghost dofs (their one local side),
      remote_src -- per owned dof, its slot in the concatenated reverse receive buffer
                    (-1: no remote side)."""

    def __init__(self, part, Lf: int, ns: int, device, scatter_src=None):
        per = Lf * ns
        self.per = per
        self.n_owned = part.n_owned_faces * per
        self.n_local = part.n_local_faces * per
        self.device = device
        i32 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int32), device=device)  # noqa: E731
        i64 = lambda a: torch.as_tensor(np.asarray(a, dtype=np.int64), device=device)  # noqa: E731
        send = {q: part.dof_index(f, Lf, ns) for q, f in sorted(part.send_faces.items())}
        recv = {q: part.dof_index(f, Lf, ns) for q, f in sorted(part.recv_faces.items())}
        # int64 copies for the torch (CPU / gloo) path
        self.send = {q: i64(i) for q, i in send.items()}
        self.recv = {q: i64(i) for q, i in recv.items()}
        self.send_counts = {q: len(i) for q, i in send.items()}
        self.recv_counts = {q: len(i) for q, i in recv.items()}
        cat = lambda d: np.concatenate([d[q] for q in sorted(d)]) if d else np.zeros(0, np.int64)  # noqa: E731
        self.fwd_send = i32(cat(send))
        self.fwd_recv = i32(cat(recv))
        remote = np.full(self.n_owned, -1, dtype=np.int64)
        o = 0
        for q in sorted(send):
            remote[send[q]] = o + np.arange(len(send[q]))
            o += len(send[q])
        self.remote_src = i32(remote)
        if scatter_src is not None:
            rs = scatter_src[cat(recv)] if len(cat(recv)) else np.zeros((0, 2), np.int64)
            if np.any(rs[:, 1] >= 0):
                raise AssertionError("a ghost trace dof with two local sides")
            self.rev_send = i32(rs[:, 0])
        else:
            self.rev_send = None
        n_s, n_r = int(self.fwd_send.numel()), int(self.fwd_recv.numel())
        f64 = lambda k: torch.empty(k, dtype=torch.float64, device=device)  # noqa: E731
        self.buf_send, self.buf_recv = f64(n_s), f64(n_r)  # forward: x out / x in
        self.rbuf_send, self.rbuf_recv = f64(n_r), f64(n_s)  # reverse: y out / y in

    # ---- kernels ----------------------------------------------------------
    def _stream(self):
        from .device import current_stream

        return current_stream()

    def _gather(self, idx, src, dst):
        _lib.check(_lib.lib().mhdg_halo_gather(idx.numel(), _lib.ptr(idx), _lib.ptr(src), _lib.ptr(dst),
                                               self._stream()), "mhdg_halo_gather")

    def _scatter(self, idx, buf, dst, accumulate):
        _lib.check(_lib.lib().mhdg_halo_scatter(idx.numel(), _lib.ptr(idx), _lib.ptr(buf), _lib.ptr(dst),
                                                int(accumulate), self._stream()), "mhdg_halo_scatter")

    # ---- forward: owned x -> local x with ghost values -----------------------
    def start_forward(self, comm, x_owned: torch.Tensor, x_local: torch.Tensor):
        """x_local[:n_owned] = x_owned and the ghost messages in flight; returns wait()
        which unpacks the ghost values (after it, x_local is complete)."""
        if not x_owned.is_cuda:  # CPU tensors: the gloo host-logic tests
            x_local[: self.n_owned] = x_owned
            got = comm.exchange({q: x_owned[i] for q, i in self.send.items()}, self.recv_counts, x_owned)
            for q, buf in got.items():
                x_local[self.recv[q]] = buf
            return lambda: None
        x_local[: self.n_owned].copy_(x_owned)
        self._gather(self.fwd_send, x_owned, self.buf_send)
        wait = _start_exchange(comm, _segments(self.buf_send, self.send_counts),
                               _segments(self.buf_recv, self.recv_counts))

        def finish():
            wait()
            self._scatter(self.fwd_recv, self.buf_recv, x_local, False)

        return finish

    def forward(self, comm: Comm, x_owned: torch.Tensor) -> torch.Tensor:
        x_local = torch.empty(self.n_local, dtype=x_owned.dtype, device=x_owned.device)
        self.start_forward(comm, x_owned, x_local)()
        return x_local

    # ---- reverse: local partial sums -> owned sums ----------------------------
    def reverse(self, comm: Comm, y_local: torch.Tensor) -> torch.Tensor:
        """Owned entries of a face-reduced local vector plus the other ranks' sides."""
        if not y_local.is_cuda:
            y_owned = y_local[: self.n_owned].clone()
            got = comm.exchange({q: y_local[i] for q, i in self.recv.items()}, self.send_counts, y_local)
            for q in sorted(got):
                y_owned.index_add_(0, self.send[q], got[q])  # unique indices per q: deterministic
            return y_owned
        self._gather(self.fwd_recv, y_local, self.rbuf_send)
        _start_exchange(comm, _segments(self.rbuf_send, self.recv_counts),
                        _segments(self.rbuf_recv, self.send_counts))()
        y_owned = y_local[: self.n_owned].clone()
        self._scatter(self.fwd_send, self.rbuf_recv, y_owned, True)
        return y_owned

    def reverse_local(self, comm: Comm, disc_c, y_loc: torch.Tensor, y_owned: torch.Tensor) -> torch.Tensor:
        """Face reduction of the unscattered local y with the reverse halo folded in
        (mhdg_face_reduce_remote): sends this rank's ghost-face sides, receives the
        other sides of its owned faces and sums both in one pass."""
        self._gather(self.rev_send, y_loc, self.rbuf_send)
        _start_exchange(comm, _segments(self.rbuf_send, self.recv_counts),
                        _segments(self.rbuf_recv, self.send_counts))()
        _lib.check(_lib.lib().mhdg_face_reduce_remote(disc_c, _lib.ptr(y_loc), _lib.ptr(self.remote_src),
                                                      _lib.ptr(self.rbuf_recv), self.n_owned, _lib.ptr(y_owned),
                                                      self._stream()), "mhdg_face_reduce_remote")
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
        self._split = None
        self._plan_device = plan_device

    @property
    def device(self):
        return self.local.device

    @property
    def plan(self) -> HaloPlan:
        if self._plan is None:
            dev = self._plan_device if self._plan_device is not None else self.local.device.device
            src = self.local.scatter_sources() if torch.device(dev).type == "cuda" else None
            self._plan = HaloPlan(self.part, self.Lf, self.ns, dev, src)
        return self._plan

    @property
    def macro_split(self):
        """(i0, i1): local macros [i0, i1) touch no ghost face (they only read owned
        trace values), the rest do.  Slabs are strips of cells, so the macros next to
        ghost faces sit at both ends of the slab's macro range."""
        if self._split is None:
            fo = self.local.mesh.faces_of_macro
            needs_ghost = (fo >= self.part.n_owned_faces).any(axis=1)
            best, i, M = (0, 0), 0, len(needs_ghost)
            while i < M:
                if needs_ghost[i]:
                    i += 1
                    continue
                j = i
                while j < M and not needs_ghost[j]:
                    j += 1
                if j - i > best[1] - best[0]:
                    best = (i, j)
                i = j
            self._split = best
        return self._split

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
        self._x_local = None

    @property
    def blocks(self):
        return self.local.blocks

    def apply_trace(self, x_owned, out=None):
        """Distributed apply (condense.py:91-103 over slabs): the forward
        halo is in flight while the macros that read only owned trace values are
        applied; the macros next to ghost faces follow once it lands; the reverse halo
        is summed inside the face reduction (mhdg_face_reduce_remote)."""
        dd, loc = self.dist, self.local
        plan = dd.plan
        if not x_owned.is_cuda:  # CPU tensors: the gloo host-logic tests
            y = dd.reverse(loc.apply_trace(dd.forward(x_owned)))
        else:
            x_owned = _lib.arg(x_owned, plan.n_owned, "x")
            if self._x_local is None:
                self._x_local = torch.empty(plan.n_local, dtype=torch.float64, device=x_owned.device)
            xl = self._x_local
            finish = plan.start_forward(self.comm, x_owned, xl)
            i0, i1 = dd.macro_split
            loc.note_applies(1)
            if loc.ahat is None and i1 > i0:
                loc.apply_trace_local_range(xl, i0, i1 - i0)  # interior: overlaps the halo
                finish()
                loc.apply_trace_local_range(xl, 0, i0)
                loc.apply_trace_local_range(xl, i1, dd.n_mac - i1)
            else:
                finish()
                loc.apply_trace_local_into(xl)
            y = torch.empty(plan.n_owned, dtype=torch.float64, device=x_owned.device)
            plan.reverse_local(self.comm, dd.local.device.c, loc._y_loc, y)
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
