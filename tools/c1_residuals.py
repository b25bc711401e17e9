import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
from paper_2402_11361_b200 import assembly as A, stepper as S, condense as CD
from paper_2402_11361_b200.cases import CouettePlane2D
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_square_mesh
g = np.load("/root/repo/tests/golden/c1_ptc_oracle.npz")
for kind in sys.argv[1:]:
    CD.FACTOR = kind
    case = CouettePlane2D()
    mesh = build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False))
    d = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10)
    print(kind, st.iterations, st.krylov_iterations, ["%.3e" % r for r in st.residuals])
print("oracle", g["newton"], g["krylov"], ["%.3e" % r for r in g["residuals"]])
