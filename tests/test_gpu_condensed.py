"""GPU parity: condensation (Schur + LU), trace apply, rhs, recover, block
preconditioner and gradient refresh against the reference's golden outputs
(3D) and the oracle restatement (2D).  Blocks come from the oracle so that
these kernels are checked independently of the assembly kernels."""

import numpy as np
import pytest
import torch

import oracle.hdg_oracle as O
from conftest import load_golden, rel_err
from golden_cases import OP_CASES, ctx_of
from gpu_util import dev, host, need_gpu, perturbed_fields, upload_blocks
from paper_2402_11361_b200 import _lib
from paper_2402_11361_b200.assembly import gradient_refresh
from paper_2402_11361_b200.cases import CouettePlane2D, UniformFlow2D
from paper_2402_11361_b200.condense import CondensedSchur
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.krylov import block_precond_build
from paper_2402_11361_b200.mesh import build_square_mesh

pytestmark = pytest.mark.gpu
TOL = 1e-10


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_condensed_ops_vs_reference(name):
    need_gpu()
    g = load_golden(name)
    d = OP_CASES[name]()
    of = O.Fields(g["u"], g["q"], g["uhat"])
    ob, _ = O.jacobian(d, of, ctx_of(g, O.Ctx))
    blocks = upload_blocks(d, ob)
    cond = CondensedSchur.allocate(blocks)
    S = host(cond.schur_matrix_into_factors())
    assert rel_err(np.einsum("mab,mb->ma", S, g["schur_probe"]), g["schur_times_probe"]) < 1e-12
    cond.refactor()
    assert rel_err(host(cond.schur_solve(dev(g["schur_probe"]))), g["schur_inv_times_probe"]) < TOL
    for x, y in zip(g["x"], g["y"]):
        assert rel_err(host(cond.apply_trace(dev(x))), y) < TOL
    res = [dev(g[k]) for k in ("R_Q", "R_U", "R_T")]
    assert rel_err(host(cond.rhs(*res)), g["rhs"]) < TOL
    du, dq = cond.recover(res[0], res[1], dev(g["x"][0]))
    assert rel_err(host(du), g["rec_du"]) < TOL
    assert rel_err(host(dq), g["rec_dq"]) < TOL
    pre = block_precond_build(cond)
    assert rel_err(host(pre(dev(g["x"][0]))), g["precond_y"]) < TOL


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_precond_build_variants_agree(name):
    """The register-tile Gauss-Jordan sweep (default) and the shared-memory Cholesky +
    triangular inverse invert the same symmetrised face blocks: inverses equal to rounding,
    and the sweep's inverse symmetric to rounding."""
    need_gpu()
    g = load_golden(name)
    d = OP_CASES[name]()
    ob, _ = O.jacobian(d, O.Fields(g["u"], g["q"], g["uhat"]), ctx_of(g, O.Ctx))
    cond = CondensedSchur.allocate(upload_blocks(d, ob))
    L = _lib.lib()
    try:
        L.mhdg_set_precond_variant(1)
        chol = block_precond_build(cond).inverse.clone()
    finally:
        L.mhdg_set_precond_variant(0)
    sweep = block_precond_build(cond).inverse
    scale = float(chol.abs().max())
    assert float((sweep - chol).abs().max()) < 1e-12 * scale
    assert float((sweep - sweep.transpose(1, 2)).abs().max()) < 1e-13 * scale
    # a face block that is not positive definite raises the reference's error class
    import dataclasses

    from paper_2402_11361_b200.krylov import PreconditionerError

    ob_bad = dataclasses.replace(ob, face_trace_trace=-np.abs(ob.face_trace_trace))
    with pytest.raises(PreconditionerError):
        block_precond_build(CondensedSchur.allocate(upload_blocks(d, ob_bad)))


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_gradient_refresh_vs_oracle(name):
    need_gpu()
    g = load_golden(name)
    d = OP_CASES[name]()
    q = gradient_refresh(d, dev(g["u"]), dev(g["uhat"]))
    assert rel_err(host(q), O.gradient_refresh(d, g["u"], g["uhat"])) < 1e-12


def _cases_2d():
    c2 = UniformFlow2D()
    c1 = CouettePlane2D()
    return {
        "uniform_m2p2": (Discretization(build_square_mesh(c2.domain, 3, 2, periodic=(True, True)), 2, c2.params),
                         c2.state, O.Ctx.steady(1.0)),
        "uniform_m4p3": (Discretization(build_square_mesh(c2.domain, 2, 4, periodic=(True, True)), 3, c2.params),
                         c2.state, O.Ctx.steady(1.0)),
        "couette_m2p2": (Discretization(build_square_mesh(c1.domain, (4, 2), 2, periodic=(True, False)), 2,
                                        c1.params, bcs=c1.boundary_conditions()), c1.exact_state, O.Ctx.steady(5.0)),
    }


@pytest.mark.parametrize("name", ["uniform_m2p2", "uniform_m4p3", "couette_m2p2"])
def test_condensed_ops_2d_vs_oracle(name):
    need_gpu()
    d, fn, ctx = _cases_2d()[name]
    of = perturbed_fields(d, fn, 7)
    res = O.residual(d, of, ctx)
    ob, _ = O.jacobian(d, of, ctx)
    oc = O.condense(ob)  # explicit inverse, as the reference
    olu = O.condense(ob, mode="lu")  # LU solves, the device's algebra
    cond = CondensedSchur.build(upload_blocks(d, ob))
    rng = np.random.default_rng(3)
    for _ in range(2):
        x = rng.standard_normal(d.n_trace)
        assert rel_err(host(cond.apply_trace(dev(x))), oc.apply_trace(x)) < TOL
    r = [dev(a) for a in res]
    b = host(cond.rhs(*r))
    # rhs = -R_T + (S^-1 of a residual): LU vs explicit inverse differ by
    # ~cond(S) eps here (cond(S) ~ 1e6 at m=4, p=3); the algebra itself is
    # pinned against the LU oracle at 1e-10.
    assert rel_err(b, olu.rhs(*res)) < TOL
    cond_s = max(np.linalg.cond(S) for S in O.schur_matrix(ob)[:4])
    assert rel_err(b, oc.rhs(*res)) < max(TOL, 100 * cond_s * np.finfo(float).eps)
    du, dq = cond.recover(r[0], r[1], dev(x))
    du0, dq0 = olu.recover(res[0], res[1], x)
    assert rel_err(host(du), du0) < TOL
    assert rel_err(host(dq), dq0) < TOL
    pre = block_precond_build(cond)
    assert rel_err(host(pre(dev(x))), O.block_precond_build(oc)(x)) < TOL


def test_apply_is_deterministic_and_linear():
    need_gpu()
    d, fn, ctx = _cases_2d()["uniform_m2p2"]
    of = perturbed_fields(d, fn, 11)
    ob, _ = O.jacobian(d, of, ctx)
    cond = CondensedSchur.build(upload_blocks(d, ob))
    rng = np.random.default_rng(5)
    x1, x2 = dev(rng.standard_normal(d.n_trace)), dev(rng.standard_normal(d.n_trace))
    y1 = cond.apply_trace(x1)
    assert torch.equal(y1, cond.apply_trace(x1))
    y12 = cond.apply_trace(2.0 * x1 - 3.0 * x2)
    assert rel_err(host(y12), host(2.0 * y1 - 3.0 * cond.apply_trace(x2))) < 1e-13


@pytest.mark.parametrize("split", [1, 0])
@pytest.mark.parametrize("name", ["uniform_m2p2", "uniform_m4p3", "couette_m2p2"])
def test_streamed_apply_matches_generic(name, split):
    """The TMA-streamed specialised kernels -- split (pre / S^-1 stream / post)
    and fused -- agree with the generic kernel."""
    need_gpu()
    from paper_2402_11361_b200 import _lib

    L = _lib.lib()
    d, fn, ctx = _cases_2d()[name]
    of = perturbed_fields(d, fn, 13)
    ob, _ = O.jacobian(d, of, ctx)
    cond = CondensedSchur.build(upload_blocks(d, ob))
    x = dev(np.random.default_rng(8).standard_normal(d.n_trace))
    try:
        L.mhdg_set_stream_enabled(0)
        y_gen = host(cond.apply_trace(x))
        L.mhdg_set_stream_enabled(1)
        L.mhdg_set_apply_split(split)
        y_str = host(cond.apply_trace(x))
        assert torch.equal(cond.apply_trace(x), cond.apply_trace(x))
    finally:
        L.mhdg_set_stream_enabled(1)
        L.mhdg_set_apply_split(1)
    assert rel_err(y_str, y_gen) < 1e-10  # summation order differs; cond(S) ~ 1e6 at m=4, p=3


@pytest.mark.parametrize("name", ["uniform_m2p2", "uniform_m4p3", "couette_m2p2"])
def test_lu_factor_kind_matches_inverse(name):
    """Packed-LU factors (k_lu4, pivots in place) and the explicit inverse give
    the same condensed operator, rhs and recovery up to cond(S) * eps."""
    need_gpu()
    from paper_2402_11361_b200 import condense as CD

    d, fn, ctx = _cases_2d()[name]
    of = perturbed_fields(d, fn, 21)
    ob, _ = O.jacobian(d, of, ctx)
    res = [dev(r) for r in O.residual(d, of, ctx)]
    blocks = upload_blocks(d, ob)
    x = dev(np.random.default_rng(3).standard_normal(d.n_trace))
    out = {}
    old = CD.FACTOR
    try:
        for kind in ("inverse", "lu"):
            CD.FACTOR = kind
            cond = CD.CondensedSchur.build(blocks)
            du, _ = cond.recover(res[0], res[1], x)
            out[kind] = (host(cond.apply_trace(x)), host(cond.rhs(*res)), host(du))
    finally:
        CD.FACTOR = old
    tol = 1e-7 if name == "uniform_m4p3" else 1e-10  # cond(S) ~ 1e6 at m=4, p=3
    for a, b in zip(out["lu"], out["inverse"]):
        assert rel_err(a, b) < tol


@pytest.mark.parametrize("m_sub,p_deg", [(1, 2), (1, 3), (4, 1)])
def test_streamed_apply_3d_m1_vs_oracle(m_sub, p_deg):
    """C5's 3D combos without a reference golden on the streamed apply: (1, 2) has an odd
    W_vol segment per macro (27 x 225 doubles), so every other macro's pieces are copied from
    one double earlier; (1, 3) exercises the point-chunked assembly; (4, 1) has 64
    sub-elements and 16 sub-faces per face (the most face-lattice sharing)."""
    need_gpu()
    from golden_cases import TGV
    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200.mesh import build_cube_mesh

    d = Discretization(build_cube_mesh(TGV.domain, 2 if m_sub == 1 else 1, m_sub, periodic=(True,) * 3), p_deg,
                       TGV.params)
    of = perturbed_fields(d, TGV.initial_state, 13)
    ob, _ = O.jacobian(d, of, O.Ctx.steady(2.0))
    gb, _ = A.jacobian(d, A.to_device_fields(d, of.u, of.q, of.uhat), A.StageContext.steady(2.0))
    for k in ("state_state", "face_trace_trace", "wdgdq_vol"):
        assert rel_err(host(getattr(gb, k)), getattr(ob, k)) < 1e-10, k
    cond, ocond = CondensedSchur.build(gb), O.condense(ob)
    rng = np.random.default_rng(5)
    with _lib.Timeline(16) as tl:
        for _ in range(3):
            x = rng.standard_normal(d.n_trace)
            assert rel_err(host(cond.apply_trace(dev(x))), ocond.apply_trace(x)) < 1e-9
    assert "apply_pre" in tl.ms and "apply_generic" not in tl.ms  # the streamed kernels ran
    cond.form_local_operators()  # stored blocks from these streamed kernels (odd W_vol segments at p = 2)
    with _lib.Timeline(16) as tl:
        for _ in range(2):
            x = rng.standard_normal(d.n_trace)
            assert rel_err(host(cond.apply_trace(dev(x))), ocond.apply_trace(x)) < 1e-9
    assert "apply_ahat" in tl.ms and "apply_pre" not in tl.ms


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_stored_local_operators_vs_reference(name):
    """B_A representation (csrc/ahat.cu): the per-macro condensed trace blocks formed
    from unit-trace local applies reproduce the reference's apply (golden y) and the
    matrix-free apply, and the blocks equal the local apply of random local traces."""
    need_gpu()
    g = load_golden(name)
    d = OP_CASES[name]()
    of = O.Fields(g["u"], g["q"], g["uhat"])
    ob, _ = O.jacobian(d, of, ctx_of(g, O.Ctx))
    cond = CondensedSchur.build(upload_blocks(d, ob))
    y_mf = [host(cond.apply_trace(dev(x))) for x in g["x"]]
    at = cond.form_local_operators()
    for x, y, ymf in zip(g["x"], g["y"], y_mf):
        y_st = host(cond.apply_trace(dev(x)))
        assert rel_err(y_st, y) < TOL
        assert rel_err(y_st, ymf) < 1e-12
    xl = torch.randn(d.n_mac, at.shape[1], dtype=torch.float64, device="cuda")
    blk = torch.einsum("mkt,mk->mt", at, xl)
    cond.ahat = None
    ident = torch.arange(d.n_mac * at.shape[1], dtype=torch.int32, device="cuda")
    # the matrix-free local apply over a local trace vector (identity gather) is the same map
    disc_c = _lib.Disc.from_buffer_copy(d.device.c)
    disc_c.gather = ident.data_ptr()
    rc = _lib.lib().mhdg_apply_trace_local(disc_c, cond.blocks.c, cond._fac, _lib.ptr(xl), _lib.ptr(cond._y_loc),
                                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    torch.cuda.synchronize()
    assert rel_err(host(cond._y_loc.view(d.n_mac, -1)), host(blk)) < 1e-12


def test_stored_local_operators_2d_c1_matches_matrix_free():
    need_gpu()
    case = CouettePlane2D()
    d = Discretization(build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False)), 2, case.params,
                       bcs=case.boundary_conditions())
    from paper_2402_11361_b200 import assembly as A
    u, uhat = d.nodal_interpolant(case.exact_state)
    fs = A.FieldState(dev(u), None, dev(uhat))
    fs.q = gradient_refresh(d, fs.u, fs.uhat)
    blocks, _ = A.jacobian(d, fs, A.StageContext.steady(1.0))
    cond = CondensedSchur.build(blocks)
    xs = [torch.randn(d.n_trace, dtype=torch.float64, device="cuda") for _ in range(3)]
    y_mf = [host(cond.apply_trace(x)) for x in xs]
    cond.form_local_operators()
    for x, ymf in zip(xs, y_mf):
        assert rel_err(host(cond.apply_trace(x)), ymf) < 1e-12
    assert torch.equal(cond.apply_trace(xs[0]), cond.apply_trace(xs[0]))


@pytest.mark.parametrize("name", ["uniform_m4p3", "couette_m2p2"])
def test_chunked_condensation_and_range_apply(name):
    """mhdg_factors.scratch_macros (Schur + LU + pack chunk by chunk) gives bitwise the
    factors of the one-shot condensation, and the local apply over macro ranges
    (mhdg_apply_trace_local_range, the slab overlap) equals the full local apply."""
    need_gpu()
    d, fn, ctx = _cases_2d()[name]
    of = perturbed_fields(d, fn, 33)
    ob, _ = O.jacobian(d, of, ctx)
    blocks = upload_blocks(d, ob)
    full = CondensedSchur.build(blocks)
    chunked = CondensedSchur.allocate(blocks, scratch_macros=3)
    assert chunked.scratch.shape[0] == 3
    chunked.refactor()
    assert torch.equal(full.lu, chunked.lu) and torch.equal(full.perm, chunked.perm)
    x = dev(np.random.default_rng(4).standard_normal(d.n_trace))
    y_full = full.apply_trace_local(x)
    for cuts in ((0, 1, d.n_mac), (0, d.n_mac // 2, d.n_mac), (0, 3, 5, d.n_mac)):
        full._y_loc.zero_()
        for a, b in zip(cuts[:-1], cuts[1:]):
            full.apply_trace_local_range(x, a, b - a)
        assert torch.equal(full._y_loc.view_as(y_full), y_full), cuts


def test_factor_size_limit_raises_config_error():
    """L ns above the factor kernels' limit (mhdg_factor_max_n) raises ConfigError at
    allocation instead of a launch failure."""
    need_gpu()
    from paper_2402_11361_b200.condense import FACTOR, FACTOR_KINDS
    from paper_2402_11361_b200.discretization import ConfigError

    n_max = int(_lib.lib().mhdg_factor_max_n(FACTOR_KINDS[FACTOR]))
    assert n_max >= 420
    c2 = UniformFlow2D()
    d = Discretization(build_square_mesh(c2.domain, 1, 8, periodic=(True, True)), 4, c2.params)  # L ns = 2244
    assert d.L * d.ns > n_max
    from paper_2402_11361_b200.assembly import LocalBlocks

    blocks = LocalBlocks.empty(d)
    with pytest.raises(ConfigError):
        CondensedSchur.allocate(blocks)
