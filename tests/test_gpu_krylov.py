"""Fused device ICGS (mhdg_icgs) vs the reference formulation (krylov.py:51-58)
evaluated with torch in float64: same projections, norm and updated vector."""

import numpy as np
import pytest
import torch

from gpu_util import need_gpu
from paper_2402_11361_b200 import krylov as K

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,j", [(37, 0), (2080, 5), (2080, 59), (638976, 20)])
def test_fused_icgs_matches_reference_formulation(n, j):
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(n + j)
    V = torch.randn(61, n, dtype=torch.float64, device="cuda", generator=g)
    V[: j + 1] = torch.linalg.qr(V[: j + 1].T)[0].T  # orthonormal basis, as in Arnoldi
    w = torch.randn(n, dtype=torch.float64, device="cuda", generator=g) + 0.5 * V[0]
    Vj = V[: j + 1]
    h = Vj @ w
    wr = w - Vj.T @ h
    h2 = Vj @ wr
    wr = wr - Vj.T @ h2
    h_ref, hv_ref = (h + h2).cpu().numpy(), float(torch.linalg.vector_norm(wr))
    h_dev, hv_dev, w_dev = K._icgs_device(V, j, w)
    assert np.abs(h_dev - h_ref).max() <= 1e-12 * max(1.0, np.abs(h_ref).max())
    assert abs(hv_dev - hv_ref) <= 1e-12 * hv_ref
    assert float((w_dev - wr).abs().max()) <= 1e-12 * float(wr.abs().max())
    # deterministic
    h_b, hv_b, w_b = K._icgs_device(V, j, w)
    assert np.array_equal(h_b, h_dev) and hv_b == hv_dev and torch.equal(w_b, w_dev)


def _c1_operator():
    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200.cases import CouettePlane2D
    from paper_2402_11361_b200.condense import CondensedSchur
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.mesh import build_square_mesh

    case = CouettePlane2D()
    d = Discretization(build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False)), 2, case.params,
                       bcs=case.boundary_conditions())
    u, uhat = d.nodal_interpolant(case.exact_state)
    rng = np.random.default_rng(0)
    u = u + rng.uniform(-1e-3, 1e-3, u.shape)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(d, f.u, f.uhat)
    blocks, _ = A.jacobian(d, f, A.StageContext.steady(1.0))
    return d, CondensedSchur.build(blocks)


@pytest.mark.parametrize("solver", ["fgmres", "gmres"])
def test_graph_captured_arnoldi_steps_are_bitwise_eager(solver, monkeypatch):
    """The CUDA-graph path of the Arnoldi steps (K._StepGraphs) replays the eager step's
    kernels on persistent buffers: same solution bit for bit, same iteration and matvec
    counts, at C1 size (BASELINE configs[0]) over several restarts."""
    need_gpu()
    d, cond = _c1_operator()
    b = torch.as_tensor(np.random.default_rng(3).standard_normal(d.n_trace), device="cuda")
    cfg = K.KrylovConfig(restart=12, max_iter=200, rel_tol=1e-9, inner_iter=6)
    runs = {}
    for on in (False, True):
        monkeypatch.setattr(K, "KRYLOV_GRAPHS", on)
        res, nmv = K.solve_trace_system(cond, b, cfg, solver)
        runs[on] = (res, nmv)
    (r0, n0), (r1, n1) = runs[False], runs[True]
    assert r0.iterations == r1.iterations and n0 == n1 and r0.converged == r1.converged
    assert torch.equal(r0.x, r1.x)
    assert r0.history == r1.history or all(
        (a[0] == c[0] and (a[1] == c[1] or (a[1] != a[1] and c[1] != c[1])) and a[2] == c[2])
        for a, c in zip(r0.history, r1.history))
    assert r0.iterations > cfg.restart  # the persistent bases are reused across restarts


def test_auto_stored_representation_mid_solve(monkeypatch):
    """MHDG_APPLY_REPR=auto: the stored local blocks are formed after ltr applies, in the
    middle of the FGMRES solve (graphs recaptured against the new apply); the solve agrees
    with the matrix-free one (iterations within 1, solution to 1e-8)."""
    need_gpu()
    from paper_2402_11361_b200 import condense as CD

    d, cond = _c1_operator()
    b = torch.as_tensor(np.random.default_rng(5).standard_normal(d.n_trace), device="cuda")
    cfg = K.KrylovConfig(rel_tol=1e-10, max_iter=400)
    r0, n0 = K.solve_trace_system(cond, b, cfg, "fgmres")
    assert cond.ahat is None
    monkeypatch.setattr(CD, "APPLY_REPR", "auto")
    cond._n_applies = 0
    r1, n1 = K.solve_trace_system(cond, b, cfg, "fgmres")
    assert cond.ahat is not None and n1 > d.nf * d.Lf * d.ns
    assert abs(r0.iterations - r1.iterations) <= 1 and r1.converged
    assert float((r1.x - r0.x).abs().max() / r0.x.abs().max()) < 1e-8


@pytest.mark.parametrize("n,rows", [(1, 1), (1000, 7), (638976, 21), (3686400, 9)])
def test_vec_pass_modes_match_torch(n, rows):
    """mhdg_vec_pass (csrc/krylov.cu), every mode, at sizes up to C3's trace length:
    dots, update + dots, update + norm, combine (x += V^T y), norm -- against torch
    float64, and bitwise deterministic."""
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(n + rows)
    V = torch.randn(rows + 1, n, dtype=torch.float64, device="cuda", generator=g)
    w0 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    c = torch.randn(rows, dtype=torch.float64, device="cuda", generator=g)
    out = torch.zeros(64, dtype=torch.float64, device="cuda")
    Vr = V[:rows]

    def run(mode):
        w = w0.clone()
        K._vec_pass(n, rows, V, w, c, mode, out)
        torch.cuda.synchronize()
        return w, out.clone()

    tol = lambda ref: 1e-12 * max(1.0, float(ref.abs().max()))  # noqa: E731
    w, o = run(0)
    assert torch.equal(w, w0) and float((o[:rows] - Vr @ w0).abs().max()) <= tol(Vr @ w0) * n ** 0.5
    upd = w0 - Vr.T @ c
    w, o = run(1)
    assert float((w - upd).abs().max()) <= tol(upd)
    assert float((o[:rows] - Vr @ upd).abs().max()) <= tol(Vr @ upd) * n ** 0.5
    w, o = run(2)
    assert abs(float(o[0]) - float(upd @ upd)) <= 1e-12 * float(upd @ upd)
    w, o = run(3)
    comb = w0 + Vr.T @ c
    assert float((w - comb).abs().max()) <= tol(comb)
    w, o = run(4)
    assert abs(float(o[0]) - float(w0 @ w0)) <= 1e-12 * float(w0 @ w0)
    for mode in range(5):  # deterministic (the outputs each mode writes)
        a, b = run(mode), run(mode)
        k = {0: rows, 1: rows, 2: 1, 3: 0, 4: 1}[mode]
        assert torch.equal(a[0], b[0]) and torch.equal(a[1][:k], b[1][:k])
