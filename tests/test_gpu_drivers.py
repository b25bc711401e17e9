"""End-to-end parity of the device Newton/FGMRES/DIRK/PTC drivers with the
reference's own runs (golden fixtures): iteration counts and converged states."""

import numpy as np
import pytest

from conftest import load_golden, rel_err
from golden_cases import COU, TGV
from gpu_util import dev, host, need_gpu
from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200 import krylov as K
from paper_2402_11361_b200 import stepper as S
from paper_2402_11361_b200.condense import condense
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_cube_mesh

pytestmark = pytest.mark.gpu


def test_krylov_solves_vs_reference():
    need_gpu()
    g = load_golden("krylov_tgv_m1p2")
    d = Discretization(build_cube_mesh(TGV.domain, 1, 1, periodic=(True,) * 3), 2, TGV.params)
    f = A.to_device_fields(d, g["u"], g["q"], g["uhat"])
    ctx = A.StageContext(50.0, dev(g["hist"]), np.inf, 0.02)
    res = A.residual(d, f, ctx)
    blocks, _ = A.jacobian(d, f, ctx)
    cond = condense(blocks)
    b = cond.rhs(*res)
    assert rel_err(host(b), g["rhs"]) < 1e-10
    for solver in ("fgmres", "gmres"):
        r, nmv = K.solve_trace_system(cond, b, K.KrylovConfig(rel_tol=1e-8), solver)
        assert r.iterations == int(g[f"{solver}_iters"])
        assert nmv == int(g[f"{solver}_matvecs"])
        assert rel_err(host(r.x), g[f"{solver}_x"]) < 1e-8


def test_dirk33_step_vs_reference():
    need_gpu()
    g = load_golden("dirk_tgv_m2p2")
    d = Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 2, TGV.params)
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    sts, _ = S.dirk_advance(d, f, float(g["dt"]), S.DirkTableau.dirk33())
    assert [s.iterations for s in sts] == list(g["newton"])
    assert all(abs(a - b) <= 1 for a, b in zip([s.krylov_iterations for s in sts], g["krylov"]))
    assert rel_err(host(f.u), g["u"]) < 1e-8
    assert rel_err(host(f.uhat), g["uhat"]) < 1e-8


def test_ptc_couette_vs_reference():
    need_gpu()
    g = load_golden("ptc_couette_m2p1")
    d = Discretization(build_cube_mesh(((0, 0, 0), (1, 1, 1)), 1, 2), 1, COU.params,
                       bcs=COU.boundary_conditions(), source=COU.source)
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10)
    assert abs(st.iterations - int(g["newton"])) <= 1
    assert abs(st.krylov_iterations - int(g["krylov"])) <= 1
    assert rel_err(host(f.u), g["u"]) < 1e-8
    assert rel_err(host(f.uhat), g["uhat"]) < 1e-8


@pytest.mark.parametrize("kind", ["lu", "inverse"])
def test_c1_plane_couette_ptc_vs_oracle(kind):
    """BASELINE configs[0] (C1) end to end on the device: PTC + FGMRES to 1e-10 from
    the seeded IC, against the oracle run with the same factor algebra
    (oracle/make_c1_golden.py: "lu" = LAPACK LU solves, "inverse" = the reference's
    explicit inverse, condense.py:67), step by step.

    Every Newton step after the first ends at FGMRES's 400-iteration cap with the
    linear system unconverged, so rounding-level differences are amplified by the
    truncated Krylov solve: the oracle's own LU and inverse runs -- solves accurate to
    1e-14 on these S -- already differ by 7e-7 in the state after step 2 and settle on
    a uniform density offset of 2.4e-7 (steady Couette between isothermal walls in a
    periodic channel leaves the density level free; PTC does not conserve mass).
    Bounds: Newton +-1; per-step FGMRES +-1 on every common step; the state after
    step 1 within 1e-8; after later common steps within 10x the oracle pair's own
    spread at that step; final temperature and velocity within max(1e-8, 10x the
    pair's spread); the final state a converged solution of the oracle's residual.  oracle/c1_ensemble.py records the
    spread of Newton counts under 1e-14 initial-state noise (profiles/r2_c1_ensemble_*)."""
    need_gpu()
    from paper_2402_11361_b200 import condense as CD
    from paper_2402_11361_b200.cases import CouettePlane2D
    from paper_2402_11361_b200.mesh import build_square_mesh
    import oracle.hdg_oracle as O

    g = load_golden("c1_ptc_oracle_lu" if kind == "lu" else "c1_ptc_oracle")
    g_other = load_golden("c1_ptc_oracle" if kind == "lu" else "c1_ptc_oracle_lu")
    case = CouettePlane2D()
    mesh = build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False))
    d = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    steps_u, steps_uhat, per_step = [], [], []

    def log(st):
        steps_u.append(host(f.u))
        steps_uhat.append(host(f.uhat))
        per_step.append(st.krylov_iterations - sum(per_step))

    old = CD.FACTOR
    try:
        CD.FACTOR = kind
        st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10, log=log)
    finally:
        CD.FACTOR = old
    print(kind, "device newton", st.iterations, "fgmres", st.krylov_iterations, per_step,
          "oracle", int(g["newton"]), int(g["krylov"]), list(g["krylov_per_step"]))
    assert abs(st.iterations - int(g["newton"])) <= 1
    common = min(st.iterations, int(g["newton"]))
    for k in range(common):
        assert abs(per_step[k] - int(g["krylov_per_step"][k])) <= 1, k
    assert abs(st.residuals[1] - g["residuals"][1]) <= 1e-8 * g["residuals"][1]  # step 1: before any cap
    for k in range(common):
        du = rel_err(steps_u[k], g["steps_u"][k])
        duh = rel_err(steps_uhat[k], g["steps_uhat"][k])
        pair = max(rel_err(g_other["steps_u"][k], g["steps_u"][k]),
                   rel_err(g_other["steps_uhat"][k], g["steps_uhat"][k]))
        print(f"  step {k + 1}: state vs oracle {du:.2e} / {duh:.2e}; oracle LU vs inverse {pair:.2e}")
        tol = 1e-8 if k == 0 else max(1e-8, 10.0 * pair)
        assert du < tol and duh < tol, (k, du, duh, pair)
    assert st.residuals[-1] <= max(1e-10, 1e-10 * st.residuals[0])  # ptc_steady_solve's target (abs_tol 1e-10)

    def prim(u):
        rho, m, E = u[..., 0], u[..., 1:3], u[..., 3]
        v = m / rho[..., None]
        T = case.gamma * (case.gamma - 1.0) * (E / rho - 0.5 * (v * v).sum(-1))
        return rho, v, T

    rho_d, v_d, T_d = prim(host(f.u))
    rho_o, v_o, T_o = prim(g["u"])
    rho_p, v_p, T_p = prim(g_other["u"])
    # the free density level leaks into v = m / rho: bound v and T by the oracle pair's
    # own final spread too (pair: 3.6e-9 in v, 2.7e-10 in T; device runs measured
    # 1.1e-8 / 1.3e-8 in v, 7.5e-10 / 9.2e-10 in T)
    for name, a, b, c in (("T", T_d, T_o, T_p), ("v", v_d, v_o, v_p)):
        e, pair = rel_err(a, b), rel_err(c, b)
        print(f"  final {name}: vs oracle {e:.2e}; oracle LU vs inverse {pair:.2e}")
        assert e < max(1e-8, 10.0 * pair), (name, e, pair)
    ratio = rho_d / rho_o  # the free density level: a uniform scale
    assert ratio.std() < 1e-8 * ratio.mean()
    of = O.Fields(host(f.u), host(f.q), host(f.uhat))
    r_dev = np.sqrt(sum(float((r * r).sum()) for r in O.residual(d, of, O.Ctx.steady())))
    assert r_dev <= 1e-10


@pytest.mark.parametrize("kind", ["lu", "inverse"])
def test_dirk33_step_with_factor_kind(kind):
    """The DIRK33 golden step with packed-LU (default) and explicit-inverse condensation factors."""
    need_gpu()
    from paper_2402_11361_b200 import condense as CD

    g = load_golden("dirk_tgv_m2p2")
    d = Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 2, TGV.params)
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    old = CD.FACTOR
    try:
        CD.FACTOR = kind
        sts, _ = S.dirk_advance(d, f, float(g["dt"]), S.DirkTableau.dirk33())
    finally:
        CD.FACTOR = old
    assert [s.iterations for s in sts] == list(g["newton"])
    assert all(abs(a - b) <= 1 for a, b in zip([s.krylov_iterations for s in sts], g["krylov"]))
    assert rel_err(host(f.u), g["u"]) < 1e-8


def test_dirk33_c3_slab_vs_reference():
    """BASELINE configs[2] (C3: TGV Re=1600, M=0.1, m=2, p=2, DIRK33, dt=0.01) on a
    2^3 x 6 = 48-macro periodic slab, two steps against the reference's own run
    (oracle/make_golden.py dirk48, stepper.py:265-328): Newton counts per stage
    equal, FGMRES within +-1 per stage, state within 1e-8 after every step."""
    need_gpu()
    g = load_golden("dirk_tgv_n2_m2p2")
    d = Discretization(build_cube_mesh(TGV.domain, 2, 2, periodic=(True,) * 3), 2, TGV.params)
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    newton, kits = [], []
    for step in range(int(g["steps"])):
        sts, dt = S.dirk_advance(d, f, float(g["dt"]), S.DirkTableau.dirk33())
        assert dt == float(g["dt"])
        newton += [s.iterations for s in sts]
        kits += [s.krylov_iterations for s in sts]
        assert rel_err(host(f.u), g["step_u"][step]) < 1e-8, step
        assert rel_err(host(f.uhat), g["step_uhat"][step]) < 1e-8, step
    assert newton == list(g["newton"])
    assert all(abs(a - b) <= 1 for a, b in zip(kits, g["krylov"]))
