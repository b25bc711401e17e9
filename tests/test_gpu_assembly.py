"""GPU parity: residuals, Jacobian blocks, stashes and frozen coefficients of
the assembly kernel against the reference's golden outputs (3D) and the
oracle restatement (2D, incl. isothermal no-slip and moving walls)."""

import numpy as np
import pytest
import torch

import oracle.hdg_oracle as O
from conftest import load_golden, rel_err
from golden_cases import OP_CASES, ctx_of
from gpu_util import dev, host, need_gpu, perturbed_fields
from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200.cases import CouettePlane2D, UniformFlow2D
from paper_2402_11361_b200.condense import condense
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_square_mesh
from paper_2402_11361_b200.physics import AdmissibilityError

pytestmark = pytest.mark.gpu
TOL = 1e-10
BLOCK_KEYS = ("state_state", "face_state_trace", "face_trace_state", "face_trace_trace", "wdgdq_vol",
              "wdgdq_face", "trace_face_scale")


def _ctx_dev(g):
    c = ctx_of(g, A.StageContext)
    if c.hist is not None:
        c.hist = dev(c.hist)
    return c


def _rq_ok(d, rq, ref, q, u=None):
    """R_Q = J M q + A_qu u + A_qh uhat cancels to ~1e-3 of its terms: compare
    at 1e-12 of the largest term."""
    scale = np.max(np.abs(O.grad_mass_apply(d, q)))
    if u is not None:
        scale = max(scale, np.max(np.abs(O.grad_state_apply(d, u))))
    return np.max(np.abs(rq - ref)) < 1e-12 * scale


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_assembly_vs_reference(name):
    need_gpu()
    g = load_golden(name)
    d = OP_CASES[name]()
    f = A.to_device_fields(d, g["u"], g["q"], g["uhat"])
    ctx = _ctx_dev(g)
    R_Q, R_U, R_T = A.residual(d, f, ctx)
    assert _rq_ok(d, host(R_Q), g["R_Q"], g["q"], g["u"])
    assert rel_err(host(R_U), g["R_U"]) < TOL
    assert rel_err(host(R_T), g["R_T"]) < TOL
    blocks, frozen = A.jacobian(d, f, ctx)
    for k in BLOCK_KEYS:
        arr = host(getattr(blocks, k))
        ref = g[f"blk_{k}"]
        assert rel_err(arr[: len(ref)], ref) < TOL, k
        assert rel_err(arr.reshape(len(arr), -1).sum(1), g[f"sum_{k}"]) < 1e-9, k
        assert rel_err(np.sqrt((arr.reshape(len(arr), -1) ** 2).sum(1)), np.sqrt(g[f"sq_{k}"])) < TOL, k
    assert rel_err(host(frozen.supg_tau), g["frz_supg_tau"]) < TOL
    assert rel_err(host(frozen.face_visc_state), g["frz_face_visc_state"]) < TOL
    # full device pipeline: assemble -> condense -> apply / rhs
    cond = condense(blocks)
    for x, y in zip(g["x"], g["y"]):
        assert rel_err(host(cond.apply_trace(dev(x))), y) < TOL
    assert rel_err(host(cond.rhs(R_Q, R_U, R_T)), g["rhs"]) < 1e-9


def _cases_2d():
    c2, c1 = UniformFlow2D(), CouettePlane2D()
    return {
        "uniform_m2p2": (Discretization(build_square_mesh(c2.domain, 3, 2, periodic=(True, True)), 2, c2.params),
                         c2.state),
        "uniform_m4p3": (Discretization(build_square_mesh(c2.domain, 2, 4, periodic=(True, True)), 3, c2.params),
                         c2.state),
        "couette_m2p2": (Discretization(build_square_mesh(c1.domain, (4, 2), 2, periodic=(True, False)), 2,
                                        c1.params, bcs=c1.boundary_conditions()), c1.exact_state),
    }


@pytest.mark.parametrize("ctx_kind", ["ptc", "dirk"])
@pytest.mark.parametrize("name", ["uniform_m2p2", "uniform_m4p3", "couette_m2p2"])
def test_assembly_2d_vs_oracle(name, ctx_kind):
    need_gpu()
    d, fn = _cases_2d()[name]
    of = perturbed_fields(d, fn, 5)
    if ctx_kind == "ptc":
        octx, gctx = O.Ctx.steady(2.0), A.StageContext.steady(2.0)
    else:
        hist = -0.7 * of.u
        octx, gctx = O.Ctx(40.0, hist, np.inf, 0.025), A.StageContext(40.0, dev(hist), np.inf, 0.025)
    f = A.to_device_fields(d, of.u, of.q, of.uhat)
    (oq, ou, ot), ob, ofz = O.assemble_system(d, of, octx)
    (gq, gu, gt), gb, gfz = A.assemble_system(d, f, gctx)
    assert _rq_ok(d, host(gq), oq, of.q, of.u)
    assert rel_err(host(gu), ou) < TOL
    assert rel_err(host(gt), ot) < TOL
    for k in BLOCK_KEYS:
        assert rel_err(host(getattr(gb, k)), getattr(ob, k)) < TOL, k
    for k in ("supg_tau", "supg_jac", "face_stab", "face_visc_state"):
        assert rel_err(host(getattr(gfz, k)), getattr(ofz, k)) < TOL, k
    # residual with frozen coefficients (finite-difference oracle mode)
    of2 = O.Fields(of.u * 1.0001, of.q, of.uhat)
    f2 = A.to_device_fields(d, of2.u, of2.q, of2.uhat)
    r_o = O.residual(d, of2, octx, frozen=ofz)
    r_g = A.residual(d, f2, gctx, frozen=gfz)
    assert rel_err(host(r_g[1]), r_o[1]) < TOL
    assert rel_err(host(r_g[2]), r_o[2]) < TOL


def test_assembly_is_deterministic():
    need_gpu()
    d, fn = _cases_2d()["couette_m2p2"]
    of = perturbed_fields(d, fn, 9)
    f = A.to_device_fields(d, of.u, of.q, of.uhat)
    ctx = A.StageContext.steady(3.0)
    r1, b1, _ = A.assemble_system(d, f, ctx)
    r2, b2, _ = A.assemble_system(d, f, ctx)
    assert all(torch.equal(a, b) for a, b in zip(r1, r2))
    assert torch.equal(b1.state_state, b2.state_state)


def test_admissibility_error():
    need_gpu()
    d, fn = _cases_2d()["uniform_m2p2"]
    of = O.interpolate(d, fn)
    u = of.u.copy()
    u[3, 5, 0] = -1.0
    f = A.to_device_fields(d, u, of.q, of.uhat)
    with pytest.raises(AdmissibilityError):
        A.residual(d, f, A.StageContext.steady())


def test_assembly_3d_p3_point_chunks_vs_oracle():
    """3D p = 3 (C5's (m, p) = (1, 3)): 64 volume points per sub-element exceed the
    kernel's shared memory in one piece, so the kernel walks them in chunks."""
    need_gpu()
    from golden_cases import TGV
    from paper_2402_11361_b200.mesh import build_cube_mesh

    d = Discretization(build_cube_mesh(TGV.domain, 1, 1, periodic=(True,) * 3), 3, TGV.params)
    of = perturbed_fields(d, TGV.initial_state, 11)
    hist = -0.7 * of.u
    octx, gctx = O.Ctx(40.0, hist, np.inf, 0.025), A.StageContext(40.0, dev(hist), np.inf, 0.025)
    f = A.to_device_fields(d, of.u, of.q, of.uhat)
    (oq, ou, ot), ob, _ = O.assemble_system(d, of, octx)
    (gq, gu, gt), gb, _ = A.assemble_system(d, f, gctx)
    assert _rq_ok(d, host(gq), oq, of.q, of.u)
    assert rel_err(host(gu), ou) < TOL
    assert rel_err(host(gt), ot) < TOL
    for k in BLOCK_KEYS:
        assert rel_err(host(getattr(gb, k)), getattr(ob, k)) < TOL, k
    cond = condense(gb)
    x = np.random.default_rng(2).standard_normal(d.n_trace)
    assert rel_err(host(cond.apply_trace(dev(x))), O.condense(ob).apply_trace(x)) < 1e-9
