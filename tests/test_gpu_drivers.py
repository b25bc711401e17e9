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
    """BASELINE configs[0] (C1) end to end on the device: PTC + FGMRES to 1e-10
    from the seeded IC, against the oracle's run (oracle/make_c1_golden.py), with the
    packed-LU (default) and explicit-inverse condensation factors."""
    need_gpu()
    from paper_2402_11361_b200 import condense as CD
    from paper_2402_11361_b200.cases import CouettePlane2D
    from paper_2402_11361_b200.mesh import build_square_mesh

    g = load_golden("c1_ptc_oracle")
    case = CouettePlane2D()
    mesh = build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False))
    d = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    old = CD.FACTOR
    try:
        CD.FACTOR = kind
        st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10)
    finally:
        CD.FACTOR = old
    # The first Newton residuals agree with the oracle's to 3 digits; from the fourth on the
    # PTC trajectory differs by the FGMRES truncation (~2% per step, in both device factor
    # kinds), so the step that crosses the 1e-10 target can move by one.  Measured: inverse
    # 8 Newton / 2879 FGMRES (oracle 8 / 2879); LU 7 / 2479 (residual 3.4e-10 -> 8.3e-11 at
    # step 7 vs the oracle's 5.6e-10 -> 1.4e-10), i.e. one Newton step and its ~400 FGMRES
    # iterations fewer.
    for a, b in zip(st.residuals[:3], g["residuals"][:3]):
        assert abs(a - b) <= 1e-3 * b
    assert abs(st.iterations - int(g["newton"])) <= 1
    if kind == "inverse":
        assert abs(st.krylov_iterations - int(g["krylov"])) <= 1
    else:
        # at most one Newton step's FGMRES iterations apart (a late PTC step takes ~400,
        # 1.25x the run's average of 360)
        per_step = 1.25 * int(g["krylov"]) / int(g["newton"])
        assert abs(st.krylov_iterations - int(g["krylov"])) <= per_step * abs(st.iterations - int(g["newton"])) + 1
    assert st.residuals[-1] <= max(1e-10, 1e-10 * st.residuals[0])  # ptc_steady_solve's target (abs_tol 1e-10)
    # Steady Couette between isothermal walls in a periodic channel fixes velocity and
    # temperature but not the pressure/density level (PTC does not conserve mass, so
    # runs land on different members of that one-parameter family): compare the
    # invariants, check the density offset is a uniform scale, and check the device
    # state is a converged solution of the oracle's own residual.
    import oracle.hdg_oracle as O

    def prim(u):
        rho, m, E = u[..., 0], u[..., 1:3], u[..., 3]
        v = m / rho[..., None]
        T = case.gamma * (case.gamma - 1.0) * (E / rho - 0.5 * (v * v).sum(-1))
        return rho, v, T

    rho_d, v_d, T_d = prim(host(f.u))
    rho_o, v_o, T_o = prim(g["u"])
    assert rel_err(T_d, T_o) < 1e-8  # measured 1.1e-9
    ratio = rho_d / rho_o  # measured: uniform offset -3.7e-7, spread 3.3e-10 (inverse), 1.0e-9 (LU:
    assert ratio.std() < 5e-9 * ratio.mean()  # stops one step earlier, residual 8.3e-11)
    # the weakly determined density level leaks into v = m / rho at the 1e-8 level (measured 1.6e-8)
    assert np.abs(v_d - v_o).max() < 5e-8 * np.abs(v_o).max()
    of = O.Fields(host(f.u), host(f.q), host(f.uhat))
    r_dev = np.sqrt(sum(float((r * r).sum()) for r in O.residual(d, of, O.Ctx.steady())))
    assert r_dev <= 1e-10  # ptc_steady_solve's target; measured 2.68e-11 (oracle run: 3.73e-11)


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
