"""Second-layer static condensation on the device (the reference's condense API).

CondensedSchur mirrors condense.py:54-127 of the reference: build() forms
S = A_uu - A_uq A_qq^-1 A_qu and factorizes it (batched LU with partial
pivoting instead of the reference's explicit np.linalg.inv, condense.py:67),
apply_trace() is the matrix-free reduced trace operator (condense.py:91-103),
rhs() and recover() the condensed right-hand side and local back-solve
(condense.py:105-127).  Vectors are torch CUDA float64 tensors in the
reference's global trace layout.
"""

from __future__ import annotations

import os

import torch

from . import _lib
from .assembly import FrozenCoeffs, LocalBlocks, RecomputeBlocks, raise_status
from .device import current_stream


# S factor kept per macro: "lu" (default: batched LU with partial pivoting, packed for
# the forward/back substitution of the apply, as BASELINE's north_star asks) or
# "inverse" (explicit S^-1 by Gauss-Jordan, what the reference's np.linalg.inv stores)
FACTOR = os.environ.get("MHDG_FACTOR", "lu")
FACTOR_KINDS = {"inverse": 0, "lu": 1}
# Trace-operator representation used by apply_trace: "matrix_free" (default: the
# reference's stored-operator algorithm, B_ref bytes per apply) or "stored" (each macro's
# condensed trace block A^{T_i}, formed once per condensation by ltr local applies, then
# one batched GEMV per apply: B_A bytes; csrc/ahat.cu) or "auto"
# (matrix-free until ltr applies have run on this condensation -- about what forming the
# blocks costs -- then stored: never more than twice the cheaper choice in hindsight) or
# "recompute" (B_min: only the S factors and the face
# preconditioner stay resident; jacobian() returns the linearisation point and the coupling
# blocks are re-formed window by window for every apply -- CondensedRecompute below)
APPLY_REPR = os.environ.get("MHDG_APPLY_REPR", "matrix_free")


class FactorizationError(RuntimeError):
    """Local factorization failed (condense.py:40-41)."""


class CondensedSchur:
    capturable = True  # apply_trace only launches kernels on the current stream (CUDA-graph safe)

    def __init__(self, blocks: LocalBlocks, lu: torch.Tensor, perm: torch.Tensor, scratch: torch.Tensor,
                 work: torch.Tensor | None = None):
        self.blocks = blocks
        self.lu = lu  # per macro: packed LU (csrc/packed_lu.cuh) or tiled S^-1 (csrc/tiled_inv.cuh)
        self.perm = perm
        self.scratch = scratch  # S before inversion
        self.work = work  # hand-off vectors of the split apply (pre -> S^-1 stream -> post)
        fac = _lib.Factors()
        fac.lu, fac.perm, fac.scratch = _lib.ptr(lu), _lib.ptr(perm), _lib.ptr(scratch)
        fac.work = _lib.ptr(work) if work is not None else None
        fac.kind = FACTOR_KINDS[FACTOR]
        fac.scratch_macros = scratch.shape[0]
        self._fac = fac
        self.ahat = None  # (n_mac, ltr, ltr) column-major local trace blocks when formed
        self._n_applies = 0
        dd = blocks.disc.device
        self._y_loc = torch.empty(dd.n_local_trace, dtype=torch.float64, device=dd.device)

    @classmethod
    def allocate(cls, blocks: LocalBlocks, scratch_macros: int | None = None) -> "CondensedSchur":
        """Factor storage for every macro; `scratch_macros` (or MHDG_CONDENSE_CHUNK) bounds
        the Schur scratch to that many macros (condensed chunk by chunk)."""
        disc = blocks.disc
        n = disc.L * disc.ns
        if scratch_macros is None:
            scratch_macros = int(os.environ.get("MHDG_CONDENSE_CHUNK", "0"))
        chunk = scratch_macros if 0 < scratch_macros < disc.n_mac else disc.n_mac
        dev = disc.device.device
        n_max = int(_lib.lib().mhdg_factor_max_n(FACTOR_KINDS[FACTOR]))
        if n > n_max:
            from .discretization import ConfigError

            raise ConfigError(f"local Schur complement size L*ns = {n} (m={disc.mesh.m}, p={disc.p}) exceeds the "
                              f"{FACTOR!r} factor kernels' limit n <= {n_max}")
        packed = int(_lib.lib().mhdg_packed_lu_size(n))
        lu = torch.empty((disc.n_mac, packed), dtype=torch.float64, device=dev)
        perm = torch.empty((disc.n_mac, n), dtype=torch.int32, device=dev)
        scratch = torch.empty((chunk, n, n), dtype=torch.float64, device=dev)
        work = torch.empty(int(_lib.lib().mhdg_apply_work_size(disc.device.c)), dtype=torch.float64, device=dev)
        return cls(blocks, lu, perm, scratch, work)

    @classmethod
    def build(cls, blocks: LocalBlocks) -> "CondensedSchur":
        self = cls.allocate(blocks)
        self.refactor()
        return self

    def refactor(self) -> None:
        """Schur complement + batched LU (mhdg_condense); raises FactorizationError."""
        dd = self.disc.device
        self._drop_representation()  # stale stored blocks must not survive a failed refactor
        status = dd.status_buffer()
        rc = _lib.lib().mhdg_condense(dd.c, self.blocks.c, self._fac, _lib.ptr(status), current_stream())
        _lib.check(rc, "mhdg_condense")
        raise_status(status, "condense")
        self._reset_representation()

    def _drop_representation(self) -> None:
        self.ahat = None
        self._n_applies = 0

    def _reset_representation(self) -> None:
        """New factors: drop stale stored blocks; form them again under MHDG_APPLY_REPR=stored."""
        self.ahat = None
        self._n_applies = 0
        if APPLY_REPR == "stored":
            self.form_local_operators()
        elif APPLY_REPR not in ("matrix_free", "auto", "recompute"):
            raise ValueError(f"MHDG_APPLY_REPR={APPLY_REPR!r}: expected 'matrix_free', 'stored', 'auto' or 'recompute'")

    def note_applies(self, k: int = 1) -> bool:
        """Count applies on this condensation; under MHDG_APPLY_REPR=auto form the stored
        blocks once ltr applies have run.  Returns True when the representation changed
        (callers holding CUDA graphs of the apply recapture).  Never forms inside a capture."""
        if torch.cuda.is_current_stream_capturing():
            return False  # a captured apply is counted when the graph replays (krylov._StepGraphs)
        self._n_applies += k
        if APPLY_REPR != "auto" or self.ahat is not None:
            return False
        disc = self.disc
        if self._n_applies < disc.nf * disc.Lf * disc.ns:
            return False
        self.form_local_operators()
        return True

    def form_local_operators(self) -> torch.Tensor:
        """Per-macro condensed trace blocks A^{T_i} (what dense_trace_operator,
        condense.py:269-291, assembles), column k = the local apply of the unit trace
        e_k; stored column-major.  Afterwards apply_trace reads these blocks only."""
        disc = self.disc
        dd = disc.device
        ltr = disc.nf * disc.Lf * disc.ns
        self.ahat = None
        at = torch.empty((disc.n_mac, ltr, ltr), dtype=torch.float64, device=dd.device)
        x_loc = torch.empty(disc.n_mac * ltr, dtype=torch.float64, device=dd.device)
        ident = torch.empty(disc.n_mac * ltr, dtype=torch.int32, device=dd.device)
        rc = _lib.lib().mhdg_ahat_form(dd.c, self.blocks.c, self._fac, _lib.ptr(at), _lib.ptr(x_loc),
                                       _lib.ptr(self._y_loc), _lib.ptr(ident), current_stream())
        _lib.check(rc, "mhdg_ahat_form")
        self.ahat = at
        return at

    def refactor_async(self, status: torch.Tensor) -> None:
        """Same as refactor() without the host synchronisation (benchmarks)."""
        dd = self.disc.device
        self._drop_representation()
        rc = _lib.lib().mhdg_condense(dd.c, self.blocks.c, self._fac, _lib.ptr(status), current_stream())
        _lib.check(rc, "mhdg_condense")
        self._reset_representation()

    @property
    def disc(self):
        return self.blocks.disc

    @property
    def factor_entries(self) -> int:
        return self.lu.numel()

    # ------------------------------------------------------------------
    def schur_matrix_into_factors(self) -> torch.Tensor:
        """Write S (unfactorized) into self.scratch and return it; for parity tests."""
        dd = self.disc.device
        if self.scratch.shape[0] != self.disc.n_mac:
            raise ValueError("schur_matrix_into_factors needs scratch for every macro (no MHDG_CONDENSE_CHUNK)")
        rc = _lib.lib().mhdg_schur_matrix(dd.c, self.blocks.c, self._fac, current_stream())
        _lib.check(rc, "mhdg_schur_matrix")
        return self.scratch

    def schur_solve(self, y: torch.Tensor) -> torch.Tensor:
        dd = self.disc.device
        y_c = _lib.arg(y, self.disc.n_mac * self.disc.L * self.disc.ns, "y")
        out = torch.empty_like(y_c)
        rc = _lib.lib().mhdg_lu_solve(dd.c, self._fac, _lib.ptr(y_c), _lib.ptr(out), current_stream())
        _lib.check(rc, "mhdg_lu_solve")
        return out

    def apply_trace(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        """Matrix-free action of the reduced trace operator (condense.py:91-103)."""
        dd = self.disc.device
        x = _lib.arg(x, self.disc.n_trace, "x")
        y = torch.empty_like(x) if out is None else out
        self.note_applies(1)
        if self.ahat is not None:
            rc = _lib.lib().mhdg_ahat_apply(dd.c, _lib.ptr(self.ahat), _lib.ptr(x), _lib.ptr(y),
                                            _lib.ptr(self._y_loc), current_stream())
            _lib.check(rc, "mhdg_ahat_apply")
            return y
        rc = _lib.lib().mhdg_apply_trace(dd.c, self.blocks.c, self._fac, _lib.ptr(x), _lib.ptr(y),
                                         _lib.ptr(self._y_loc), current_stream())
        _lib.check(rc, "mhdg_apply_trace")
        return y

    def apply_trace_local_into(self, x: torch.Tensor) -> None:
        """Unscattered local apply of all macros into the scratch y_loc (no copy)."""
        dd = self.disc.device
        x = _lib.arg(x, self.disc.n_trace, "x")
        if self.ahat is not None:
            rc = _lib.lib().mhdg_ahat_apply_local(dd.c, _lib.ptr(self.ahat), _lib.ptr(x), _lib.ptr(self._y_loc),
                                                  current_stream())
        else:
            rc = _lib.lib().mhdg_apply_trace_local(dd.c, self.blocks.c, self._fac, _lib.ptr(x),
                                                   _lib.ptr(self._y_loc), current_stream())
        _lib.check(rc, "mhdg_apply_trace_local")

    def apply_trace_local_range(self, x: torch.Tensor, mac0: int, count: int) -> None:
        """Matrix-free local apply of macros [mac0, mac0 + count) into y_loc (the
        slab's interior / halo-adjacent split, dist.DistCondensed.apply_trace)."""
        if count <= 0:
            return
        dd = self.disc.device
        rc = _lib.lib().mhdg_apply_trace_local_range(dd.c, self.blocks.c, self._fac, _lib.ptr(x),
                                                     _lib.ptr(self._y_loc), int(mac0), int(count), current_stream())
        _lib.check(rc, "mhdg_apply_trace_local_range")

    def apply_trace_local(self, x: torch.Tensor) -> torch.Tensor:
        dd = self.disc.device
        x = _lib.arg(x, self.disc.n_trace, "x")
        if self.ahat is not None:
            rc = _lib.lib().mhdg_ahat_apply_local(dd.c, _lib.ptr(self.ahat), _lib.ptr(x), _lib.ptr(self._y_loc),
                                                  current_stream())
        else:
            rc = _lib.lib().mhdg_apply_trace_local(dd.c, self.blocks.c, self._fac, _lib.ptr(x),
                                                   _lib.ptr(self._y_loc), current_stream())
        _lib.check(rc, "mhdg_apply_trace_local")
        return self._y_loc.view(self.disc.n_mac, self.disc.nf, self.disc.Lf, self.disc.ns).clone()

    def rhs(self, res_grad, res_state, res_trace) -> torch.Tensor:
        dd = self.disc.device
        disc = self.disc
        nu = disc.n_mac * disc.L * disc.ns
        rg = _lib.arg(res_grad, nu * disc.dim, "R_Q")  # bound locals: alive across the call
        ru = _lib.arg(res_state, nu, "R_U")
        rt = _lib.arg(res_trace, disc.n_trace, "R_T")
        b = torch.empty(disc.n_trace, dtype=torch.float64, device=dd.device)
        rc = _lib.lib().mhdg_condensed_rhs(dd.c, self.blocks.c, self._fac, _lib.ptr(rg), _lib.ptr(ru), _lib.ptr(rt),
                                           _lib.ptr(b), _lib.ptr(self._y_loc), current_stream())
        _lib.check(rc, "mhdg_condensed_rhs")
        return b

    def recover(self, res_grad, res_state, dtrace):
        disc = self.disc
        dev = disc.device.device
        du = torch.empty((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device=dev)
        dq = torch.empty((disc.n_mac, disc.dim, disc.L, disc.ns), dtype=torch.float64, device=dev)
        nu = disc.n_mac * disc.L * disc.ns
        rg = _lib.arg(res_grad, nu * disc.dim, "R_Q")  # bound locals: alive across the call
        ru = _lib.arg(res_state, nu, "R_U")
        dt = _lib.arg(dtrace, disc.n_trace, "dtrace")
        rc = _lib.lib().mhdg_recover(disc.device.c, self.blocks.c, self._fac, _lib.ptr(rg), _lib.ptr(ru),
                                     _lib.ptr(dt), _lib.ptr(du), _lib.ptr(dq), current_stream())
        _lib.check(rc, "mhdg_recover")
        return du, dq


class CondensedRecompute(CondensedSchur):
    """CondensedSchur under the coupling-recompute representation (B_min; PAPER.md:550
    "store only S^-1 and transformation data"): per macro only the packed
    LU of S, its pivots and the hand-off vectors stay resident -- (L ns)^2 + O(L ns)
    doubles -- next to the linearisation point (u, q, uhat).  build() walks the macros in
    windows of `blocks.chunk`: assemble the window's Jacobian blocks, form and factor S
    into its whole-mesh slot, add the window's trace-trace blocks to the per-face
    preconditioner sums.  apply_trace / rhs / recover re-form a window's coupling blocks
    (mhdg_assemble_window, want_jac = 2: face blocks and dG/dq stashes only) right before
    the window's local kernels read them, so the data the apply streams from HBM per
    macro drops from B_ref to about B_min plus the window buffer's L2-resident traffic,
    at the price of the pointwise Jacobians per apply.  Results are those of
    CondensedSchur bit for bit (same kernels on the same block values)."""

    capturable = True

    def __init__(self, blocks: RecomputeBlocks, precond: bool = True):
        disc = blocks.disc
        n = disc.L * disc.ns
        dev = disc.device.device
        self._with_precond = precond  # False: the face preconditioner is built when first asked for
        n_max = int(_lib.lib().mhdg_factor_max_n(FACTOR_KINDS[FACTOR]))
        if n > n_max:
            from .discretization import ConfigError

            raise ConfigError(f"local Schur complement size L*ns = {n} exceeds the {FACTOR!r} factor kernels' "
                              f"limit n <= {n_max}")
        packed = int(_lib.lib().mhdg_packed_lu_size(n))
        lu = torch.empty((disc.n_mac, packed), dtype=torch.float64, device=dev)
        perm = torch.empty((disc.n_mac, n), dtype=torch.int32, device=dev)
        scratch = torch.empty((blocks.chunk, n, n), dtype=torch.float64, device=dev)
        work = torch.empty(int(_lib.lib().mhdg_apply_work_size(disc.device.c)), dtype=torch.float64, device=dev)
        super().__init__(blocks, lu, perm, scratch, work)
        self.window = None  # coupling blocks of one window (no state_state)
        self.precond_inverse = None

    @classmethod
    def build(cls, blocks: RecomputeBlocks, precond: bool = True) -> "CondensedRecompute":
        self = cls(blocks, precond)
        self.refactor()
        return self

    def _windows(self):
        M, C = self.disc.n_mac, self.blocks.chunk
        return [(m0, min(C, M - m0)) for m0 in range(0, M, C)]

    def refactor(self) -> None:
        rb, disc = self.blocks, self.disc
        dd = disc.device
        dev, C, d, n = dd.device, rb.chunk, disc.dim, disc.L * disc.ns
        bs = disc.Lf * disc.ns
        self.window = self.precond_inverse = None
        win = LocalBlocks.empty(disc, n_mac=C)
        fro = FrozenCoeffs.empty(disc, n_mac=C)
        z = lambda k: torch.empty(k, dtype=torch.float64, device=dev)  # noqa: E731
        res = (z(C * d * n), z(C * n), z(C * disc.nf * bs))
        sums = None
        if self._with_precond:
            sums = torch.zeros((disc.mesh.n_faces, bs, bs), dtype=torch.float64, device=dev)
        status = dd.status_buffer()
        L, st = _lib.lib(), current_stream()
        for m0, cnt in self._windows():
            rb.assemble_window(m0, cnt, 1, win, status, frozen=fro, res=res)
            _lib.check(L.mhdg_condense_window(dd.c, win.c, self._fac, m0, cnt, _lib.ptr(status), st),
                       "mhdg_condense_window")
            if sums is not None:
                _lib.check(L.mhdg_face_sum_window(dd.c, win.c, _lib.ptr(sums), m0, cnt, st), "mhdg_face_sum_window")
        raise_status(status, "condense")
        del fro, res
        if sums is not None:
            self._invert_face_sums(sums)
        del sums
        self.window = LocalBlocks(disc, **{k: (None if k == "state_state" else getattr(win, k))
                                           for k in LocalBlocks.KEYS})
        del win
        self._n_applies = 0

    def refactor_async(self, status: torch.Tensor) -> None:
        raise NotImplementedError("the coupling-recompute representation condenses window by window (refactor())")

    def _invert_face_sums(self, sums: torch.Tensor) -> None:
        dd = self.disc.device
        status = dd.status_buffer()
        inv = torch.empty_like(sums)
        _lib.check(_lib.lib().mhdg_precond_build_sums(dd.c, _lib.ptr(sums), _lib.ptr(inv), _lib.ptr(status),
                                                      current_stream()), "mhdg_precond_build_sums")
        self._precond_status = status  # checked when the preconditioner is asked for (krylov.py:194-238)
        self.precond_inverse = inv

    def block_precond_build(self):
        from .krylov import BlockPreconditioner

        if self.precond_inverse is None:  # built lazily: one couplings pass for the trace-trace blocks
            disc = self.disc
            bs = disc.Lf * disc.ns
            sums = torch.zeros((disc.mesh.n_faces, bs, bs), dtype=torch.float64, device=disc.device.device)
            L, st = _lib.lib(), current_stream()
            self._local(lambda m0, cnt: _lib.check(
                L.mhdg_face_sum_window(disc.device.c, self.window.c, _lib.ptr(sums), m0, cnt, st),
                "mhdg_face_sum_window"))
            self._invert_face_sums(sums)
        raise_status(self._precond_status, "precond_build")
        return BlockPreconditioner(self, inverse=self.precond_inverse)

    def note_applies(self, k: int = 1) -> bool:
        if not torch.cuda.is_current_stream_capturing():
            self._n_applies += k
        return False

    def form_local_operators(self):
        raise NotImplementedError("stored local operators need resident blocks (MHDG_APPLY_REPR=stored)")

    def schur_matrix_into_factors(self):
        raise NotImplementedError("S is formed and factored window by window under the recompute representation")

    def _local(self, call) -> None:
        """Re-form each window's couplings, then run `call(m0, cnt)` on it (stream order
        keeps the one window buffer consistent)."""
        status = None  # the linearisation point was admissible when the factors were built
        for m0, cnt in self._windows():
            self.blocks.assemble_window(m0, cnt, 2, self.window, status)
            call(m0, cnt)

    def apply_trace_local_into(self, x: torch.Tensor) -> None:
        dd = self.disc.device
        x = _lib.arg(x, self.disc.n_trace, "x")
        L, st = _lib.lib(), current_stream()
        self._local(lambda m0, cnt: _lib.check(
            L.mhdg_apply_trace_local_window(dd.c, self.window.c, self._fac, _lib.ptr(x), _lib.ptr(self._y_loc),
                                            m0, cnt, st), "mhdg_apply_trace_local_window"))

    def apply_trace(self, x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        x = _lib.arg(x, self.disc.n_trace, "x")
        y = torch.empty_like(x) if out is None else out
        self.note_applies(1)
        self.apply_trace_local_into(x)
        _lib.check(_lib.lib().mhdg_face_reduce(self.disc.device.c, _lib.ptr(self._y_loc), _lib.ptr(y),
                                               current_stream()), "mhdg_face_reduce")
        return y

    def apply_trace_local(self, x: torch.Tensor) -> torch.Tensor:
        self.apply_trace_local_into(x)
        return self._y_loc.view(self.disc.n_mac, self.disc.nf, self.disc.Lf, self.disc.ns).clone()

    def apply_trace_local_range(self, x, mac0, count):
        raise NotImplementedError("slab ranges are not combined with the recompute representation")

    def rhs(self, res_grad, res_state, res_trace) -> torch.Tensor:
        disc = self.disc
        dd = disc.device
        nu = disc.n_mac * disc.L * disc.ns
        rg = _lib.arg(res_grad, nu * disc.dim, "R_Q")
        ru = _lib.arg(res_state, nu, "R_U")
        rt = _lib.arg(res_trace, disc.n_trace, "R_T")
        b = torch.empty(disc.n_trace, dtype=torch.float64, device=dd.device)
        L, st = _lib.lib(), current_stream()
        self._local(lambda m0, cnt: _lib.check(
            L.mhdg_condensed_rhs_local_window(dd.c, self.window.c, self._fac, _lib.ptr(rg), _lib.ptr(ru),
                                              _lib.ptr(self._y_loc), m0, cnt, st), "mhdg_condensed_rhs_local_window"))
        _lib.check(L.mhdg_face_reduce_axpy(dd.c, _lib.ptr(self._y_loc), _lib.ptr(rt), -1.0, _lib.ptr(b), st),
                   "mhdg_face_reduce_axpy")
        return b

    def recover(self, res_grad, res_state, dtrace):
        disc = self.disc
        dd = disc.device
        du = torch.empty((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device=dd.device)
        dq = torch.empty((disc.n_mac, disc.dim, disc.L, disc.ns), dtype=torch.float64, device=dd.device)
        nu = disc.n_mac * disc.L * disc.ns
        rg = _lib.arg(res_grad, nu * disc.dim, "R_Q")
        ru = _lib.arg(res_state, nu, "R_U")
        dt = _lib.arg(dtrace, disc.n_trace, "dtrace")
        L, st = _lib.lib(), current_stream()
        self._local(lambda m0, cnt: _lib.check(
            L.mhdg_recover_window(dd.c, self.window.c, self._fac, _lib.ptr(rg), _lib.ptr(ru), _lib.ptr(dt),
                                  _lib.ptr(du), _lib.ptr(dq), m0, cnt, st), "mhdg_recover_window"))
        return du, dq


def condense(blocks: LocalBlocks, path: str = "schur") -> CondensedSchur:
    """condense.py:261-266; only the second-layer path runs on the device (the
    one-shot 'standard' path is a CPU oracle in the reference)."""
    if path != "schur":
        raise ValueError(f"unknown condensation path {path!r} (the device path is 'schur')")
    if getattr(blocks, "dist", None) is not None:
        from .dist import condense_distributed

        return condense_distributed(blocks, path)
    if isinstance(blocks, RecomputeBlocks):
        return CondensedRecompute.build(blocks)
    return CondensedSchur.build(blocks)
