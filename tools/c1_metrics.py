import sys; sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
import oracle.hdg_oracle as O
from conftest import load_golden
from paper_2402_11361_b200 import assembly as A, stepper as S
from paper_2402_11361_b200.cases import CouettePlane2D
from paper_2402_11361_b200.mesh import build_square_mesh
from paper_2402_11361_b200.discretization import Discretization
g = load_golden("c1_ptc_oracle")
case = CouettePlane2D()
mesh = build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False))
d = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10)
def prim(u):
    rho, m, E = u[..., 0], u[..., 1:3], u[..., 3]
    v = m / rho[..., None]
    T = case.gamma * (case.gamma - 1.0) * (E / rho - 0.5 * (v * v).sum(-1))
    return rho, v, T
ud = f.u.cpu().numpy()
rd, vd, Td = prim(ud); ro, vo, To = prim(g["u"])
print("newton", st.iterations, g["newton"], "krylov", st.krylov_iterations, g["krylov"], "res", st.residuals[-1], g["residuals"][-1])
print("u rel", np.abs(ud-g["u"]).max()/np.abs(g["u"]).max())
print("v abs", np.abs(vd-vo).max(), "v rel to scale", np.abs(vd-vo).max()/np.abs(vo).max())
print("T rel", np.abs(Td-To).max()/np.abs(To).max())
ratio = rd/ro; print("rho ratio mean", ratio.mean()-1, "std", ratio.std())
of = O.Fields(ud, f.q.cpu().numpy(), f.uhat.cpu().numpy())
print("oracle residual at device state", np.sqrt(sum(float((r*r).sum()) for r in O.residual(d, of, O.Ctx.steady()))))
og = O.Fields(g["u"], g["q"], g["uhat"])
print("oracle residual at oracle state", np.sqrt(sum(float((r*r).sum()) for r in O.residual(d, og, O.Ctx.steady()))))
