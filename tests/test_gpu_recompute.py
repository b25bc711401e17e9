"""Coupling-recompute representation (B_min): only
the S factors stay resident and the coupling blocks are re-formed window by window.
It runs the same kernels on the same block values as the resident representation, so
everything is compared bitwise: the couplings-only assembly against the full
assembly, the window-built factors, pivots and preconditioner, apply / rhs / recover
(uneven windows), and a DIRK33 step of the 3D TGV driven through the unchanged
stepper with MHDG_APPLY_REPR=recompute."""

import numpy as np
import pytest
import torch

from gpu_util import need_gpu
from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200 import krylov as K
from paper_2402_11361_b200 import stepper as S
from paper_2402_11361_b200.condense import CondensedRecompute, CondensedSchur, condense

pytestmark = pytest.mark.gpu


def _tgv(n_ele=2, m=2, p=2):
    from paper_2402_11361_b200.cases import TgvCase
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.mesh import build_cube_mesh

    case = TgvCase(reynolds=1600.0, mach=0.1)
    disc = Discretization(build_cube_mesh(case.domain, n_ele, m, periodic=(True, True, True)), p, case.params)
    f = A.interpolate(disc, case.initial_state)
    g = torch.Generator(device="cuda").manual_seed(3)
    hist = 1e-2 * torch.randn(f.u.shape, dtype=torch.float64, device="cuda", generator=g)
    return disc, f, A.StageContext(50.0, hist, np.inf, 0.02)


def _c2_patch():
    from paper_2402_11361_b200.cases import UniformFlow2D
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.mesh import build_square_mesh

    case = UniformFlow2D()
    disc = Discretization(build_square_mesh(case.domain, 8, 4, periodic=(True, True)), 3, case.params)
    u, uhat = disc.nodal_interpolant(case.state)
    rng = np.random.default_rng(0)
    u = u + rng.normal(0.0, 1e-2, u.shape)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    return disc, f, A.StageContext.steady(1.0)


@pytest.fixture
def couplings_kernel(request):
    """The couplings-only assembly: the dedicated k_couplings kernel (1, default) or
    k_assemble's Jacobian path with the state_state work skipped (0)."""
    from paper_2402_11361_b200 import _lib

    _lib.lib().mhdg_set_couplings_kernel(request.param)
    yield request.param
    _lib.lib().mhdg_set_couplings_kernel(1)


@pytest.mark.parametrize("couplings_kernel", [1, 0], indirect=True)
@pytest.mark.parametrize("cfg,chunk", [("tgv", 20), ("tgv", 48), ("c2", 48), ("tgv13", 7)])
def test_recompute_equals_resident_bitwise(cfg, chunk, couplings_kernel):
    need_gpu()
    disc, f, ctx = _c2_patch() if cfg == "c2" else (_tgv(1, 1, 3) if cfg == "tgv13" else _tgv())
    res = A.residual(disc, f, ctx)
    blocks, _ = A.jacobian(disc, f, ctx, recompute=False)
    ref = CondensedSchur.build(blocks)
    rb = A.RecomputeBlocks(disc, f, ctx, chunk=chunk)
    cond = condense(rb)
    assert isinstance(cond, CondensedRecompute) and cond.window.state_state is None
    assert torch.equal(cond.lu, ref.lu) and torch.equal(cond.perm, ref.perm)
    # the couplings-only assembly of the last window = the full assembly's blocks
    m0, cnt = cond._windows()[-1]
    for k in blocks.KEYS:
        if k != "state_state":
            assert torch.equal(getattr(cond.window, k)[:cnt], getattr(blocks, k)[m0:m0 + cnt]), k
    g = torch.Generator(device="cuda").manual_seed(11)
    x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda", generator=g)
    assert torch.equal(cond.apply_trace(x), ref.apply_trace(x))
    assert torch.equal(cond.apply_trace_local(x), ref.apply_trace_local(x))
    assert torch.equal(cond.rhs(*res), ref.rhs(*res))
    du, dq = cond.recover(res[0], res[1], x)
    du0, dq0 = ref.recover(res[0], res[1], x)
    assert torch.equal(du, du0) and torch.equal(dq, dq0)
    pre, pre0 = cond.block_precond_build(), K.block_precond_build(ref)
    assert torch.equal(pre.inverse, pre0.inverse)
    assert torch.equal(pre(x), pre0(x))
    # the preconditioner built lazily from a couplings pass (CondensedRecompute.build(precond=False))
    lazy = CondensedRecompute.build(rb, precond=False)
    assert lazy.precond_inverse is None
    assert torch.equal(lazy.block_precond_build().inverse, pre0.inverse)


def test_dirk33_step_with_recompute_representation(monkeypatch):
    need_gpu()
    disc, f, _ = _tgv()
    f2 = f.copy()
    cfg = K.KrylovConfig()
    st_ref, _ = S.dirk_advance(disc, f, 0.01, S.DirkTableau.dirk33(), krylov_cfg=cfg)
    monkeypatch.setenv("MHDG_APPLY_REPR", "recompute")
    monkeypatch.setenv("MHDG_RECOMPUTE_CHUNK", "20")
    st, _ = S.dirk_advance(disc, f2, 0.01, S.DirkTableau.dirk33(), krylov_cfg=cfg)
    assert [s.iterations for s in st] == [s.iterations for s in st_ref]
    assert [s.krylov_iterations for s in st] == [s.krylov_iterations for s in st_ref]
    assert [s.krylov_matvecs for s in st] == [s.krylov_matvecs for s in st_ref]
    assert torch.equal(f2.u, f.u) and torch.equal(f2.q, f.q) and torch.equal(f2.uhat, f.uhat)
