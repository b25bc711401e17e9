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
