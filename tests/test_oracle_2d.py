"""CPU checks of the 2D generalisation of the reference algebra (the
reference is 3D-only, so 2D parity is pinned by internal consistency):
free-stream preservation, matrix-free condensed operator == dense one-shot
elimination, and central finite differences of every Jacobian block (frozen
coefficients, as the reference's FD oracle, assembly.py:84-96)."""

import numpy as np
import pytest

import oracle.hdg_oracle as O
from conftest import rel_err
from paper_2402_11361_b200.cases import CouettePlane2D, UniformFlow2D
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_square_mesh, count_dofs


def _uniform(n=2, m=2, p=2):
    c = UniformFlow2D()
    return c, Discretization(build_square_mesh(c.domain, n, m, periodic=(True, True)), p, c.params)


def _couette(nx=2, ny=1, m=2, p=1):
    c = CouettePlane2D()
    return c, Discretization(build_square_mesh(c.domain, (nx, ny), m, periodic=(True, False)), p, c.params,
                             bcs=c.boundary_conditions())


def test_free_stream_2d():
    c, d = _uniform(3, 2, 2)
    f = O.interpolate(d, c.state)
    for ctx in (O.Ctx.steady(), O.Ctx.steady(2.0)):
        R_Q, R_U, R_T = O.residual(d, f, ctx)
        assert np.max(np.abs(R_U)) < 1e-12 * np.max(np.abs(f.u))
        assert np.max(np.abs(R_T)) < 1e-12 * np.max(np.abs(f.u))
        assert np.max(np.abs(R_Q)) < 1e-12 * np.max(np.abs(f.u))


def test_dof_counts_2d():
    _, d = _uniform(4, 4, 3)
    tot, tr, per = count_dofs(d.mesh, 3)
    assert per == 4 * 3 * 91 and tr == 4 * d.mesh.n_faces * 13 and tot == d.n_mac * per
    assert d.mesh.n_faces == 3 * d.n_mac // 2  # fully periodic triangulation


@pytest.mark.parametrize("case", ["uniform", "couette"])
def test_matrix_free_equals_dense_2d(case):
    c, d = _uniform(2, 2, 1) if case == "uniform" else _couette(2, 1, 2, 1)
    fn = c.state if case == "uniform" else c.exact_state
    f = O.interpolate(d, fn)
    f.u = f.u * (1.0 + 1e-3 * np.random.default_rng(0).standard_normal(f.u.shape))
    blocks, _ = O.jacobian(d, f, O.Ctx.steady(3.0))
    cond = O.condense(blocks)
    A = O.dense_trace_operator(blocks)
    rng = np.random.default_rng(1)
    for _ in range(3):
        x = rng.standard_normal(d.n_trace)
        assert rel_err(cond.apply_trace(x), A @ x) < 1e-11


def _fd(fun, x, dx, eps):
    return (fun(x + eps * dx) - fun(x - eps * dx)) / (2 * eps)


@pytest.mark.parametrize("case", ["uniform", "couette"])
def test_jacobian_blocks_finite_differences_2d(case):
    """Each block vs central FD of the residual with frozen coefficients."""
    c, d = _uniform(2, 2, 2) if case == "uniform" else _couette(2, 1, 2, 2)
    fn = c.state if case == "uniform" else c.exact_state
    f = O.interpolate(d, fn)
    rng = np.random.default_rng(4)
    f.u = f.u * (1.0 + 1e-3 * rng.standard_normal(f.u.shape))
    f.uhat = f.uhat * (1.0 + 1e-3 * rng.standard_normal(f.uhat.shape))
    ctx = O.Ctx(5.0, -0.2 * f.u, np.inf, 0.05)
    blocks, frozen = O.jacobian(d, f, ctx)
    M, L, ns = d.n_mac, d.L, d.ns

    def R(u, q, uh):
        return O.residual(d, O.Fields(u, q, uh), ctx, frozen=frozen)

    du = rng.standard_normal(f.u.shape) * np.abs(f.u).max() * 1e-2
    dq = rng.standard_normal(f.q.shape) * 1e-2
    dh = rng.standard_normal(f.uhat.shape) * np.abs(f.uhat).max() * 1e-2
    eps = 1e-4
    # d/dU
    fdU = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u + s * du, f.q, f.uhat)[1:]]), 0.0, 1.0, eps)
    jU = np.einsum("mab,mb->ma", blocks.state_state, du.reshape(M, -1)).ravel()
    n_u = jU.size
    assert rel_err(jU, fdU[:n_u]) < 1e-6
    jT = O.scatter_add(d, O.trace_state_apply(blocks, du))
    assert rel_err(jT, fdU[n_u:]) < 1e-6
    # d/dQ
    fdQ = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u, f.q + s * dq, f.uhat)[1:]]), 0.0, 1.0, eps)
    assert rel_err(O.state_grad_apply(blocks, dq).ravel(), fdQ[:n_u]) < 1e-6
    assert rel_err(O.scatter_add(d, O.trace_grad_apply(blocks, dq)), fdQ[n_u:]) < 1e-6
    # d/dUhat
    fdH = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u, f.q, f.uhat + s * dh)[1:]]), 0.0, 1.0, eps)
    xl = O.gather_local(d, dh)
    assert rel_err(O.state_trace_apply(blocks, xl).ravel(), fdH[:n_u]) < 1e-6
    assert rel_err(O.scatter_add(d, O.trace_trace_apply(blocks, xl)), fdH[n_u:]) < 1e-6
    # the gradient equation is linear: its blocks are exact
    fdQQ = _fd(lambda s: R(f.u, f.q + s * dq, f.uhat)[0].ravel(), 0.0, 1.0, 1.0)
    assert rel_err(O.grad_mass_apply(d, dq).ravel(), fdQQ) < 1e-10
