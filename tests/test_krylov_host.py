"""Host-side Krylov logic on CPU tensors (no GPU): GMRES / FGMRES orchestration of
krylov.py (reference krylov.py:61-191) on a dense operator against a direct solve, the
matvec counter, and the gating of the CUDA-graph path (`_step_graphs`)."""

from types import SimpleNamespace

import numpy as np
import torch

from paper_2402_11361_b200 import krylov as K


def _system(n=80, seed=0):
    rng = np.random.default_rng(seed)
    A = np.eye(n) * 4.0 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    return torch.as_tensor(A), torch.as_tensor(b), np.linalg.solve(A, b)


def test_gmres_and_fgmres_converge_to_direct_solve():
    A, b, xs = _system()
    op = lambda v: A @ v  # noqa: E731
    cfg = K.KrylovConfig(restart=10, max_iter=200, rel_tol=1e-12, abs_tol=1e-14)
    r = K.gmres(op, b, cfg=cfg)
    assert r.converged and r.iterations > 10  # restarted at least once
    assert np.abs(r.x.numpy() - xs).max() < 1e-9 * np.abs(xs).max()
    inner = lambda v: K.gmres(op, v, cfg=K.KrylovConfig(restart=4, max_iter=4, rel_tol=0.1)).x  # noqa: E731
    rf = K.fgmres(op, b, inner, cfg=cfg)
    assert rf.converged and rf.iterations < r.iterations
    assert np.abs(rf.x.numpy() - xs).max() < 1e-9 * np.abs(xs).max()


def test_counted_operator_and_graph_gating():
    A, b, _ = _system(32)
    op, count = K.make_counted(lambda v: A @ v, capturable=True)
    K.gmres(op, b, cfg=K.KrylovConfig(restart=5, max_iter=5, rel_tol=1e-30, abs_tol=1e-300))
    assert count["n"] == 5 + 1  # 5 Arnoldi steps + the true residual of the cycle
    cfg = K.KrylovConfig(restart=5)
    assert K._step_graphs(op, None, "gmres", cfg, b, None) is None  # CPU vectors: eager path
    plain, _ = K.make_counted(lambda v: A @ v)
    assert not plain.capturable and plain.graph_ws == {}
    comm = SimpleNamespace(world=2)
    assert K._step_graphs(op, None, "gmres", cfg, b, comm) is None  # distributed: eager path
