"""C4 golden fixture from the oracle (test infrastructure).  The reference can
run neither the O-grid nor the adiabatic wall, so C4 parity rests
on the oracle restatement: its 3D algebra is pinned to the reference by
tests/test_oracle_golden.py and the new wall rows by the finite-difference
checks in tests/test_sphere.py.

Reduced C4 (BASELINE configs[3] at test size): O-grid 2 radial (grading 1.15,
r = 0.5 .. 3) x 3 polar x 4 azimuthal cells, Kuhn split, pole wedges -> 96
macros, m = 2, p = 1; Re = 100, M = 0.2; adiabatic no-slip sphere, free-stream
far field; IC free stream plus U(-1e-3, 1e-3) on every U and U-hat coefficient
(default_rng(0)), q = gradient_refresh; 5 PTC Newton steps (tau_init 1) with
FGMRES, as the C4 workload.  Writes tests/golden/sphere_ptc_oracle.npz.

    python oracle/make_sphere_golden.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle.hdg_oracle as O  # noqa: E402
from paper_2402_11361_b200.cases import SphereCase  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_sphere_ogrid_mesh  # noqa: E402

NEWTON_STEPS = 5


def sphere_setup(n_r=2, n_theta=3, n_phi=4, m=2, p=1, r_out=3.0, seed=0):
    case = SphereCase()
    mesh = build_sphere_ogrid_mesh(n_r, n_theta, n_phi, m, r_out=r_out)
    disc = Discretization(mesh, p, case.params, bcs=case.boundary_conditions())
    u, uhat = disc.nodal_interpolant(case.freestream)
    rng = np.random.default_rng(seed)
    u = u + rng.uniform(-1e-3, 1e-3, u.shape)
    uhat = uhat + rng.uniform(-1e-3, 1e-3, uhat.shape)
    return case, disc, u, uhat


def main():
    case, disc, u, uhat = sphere_setup()
    q = O.gradient_refresh(disc, u, uhat)
    f = O.Fields(u.copy(), q.copy(), uhat.copy())
    ptc = O.PtcState(dtau=1.0, tau_init=1.0, tau_max=1e8)
    t0 = time.perf_counter()
    st = O.newton_solve(disc, f, O.Ctx.steady(), max_newton=NEWTON_STEPS, ptc=ptc, abs_tol=1e-10, rel_tol=1e-10)
    dt = time.perf_counter() - t0
    out = os.path.join(ROOT, "tests", "golden", "sphere_ptc_oracle.npz")
    np.savez_compressed(out, u0=u, q0=q, uhat0=uhat, u=f.u, q=f.q, uhat=f.uhat, newton=st.iterations,
                        krylov=st.krylov_iterations, residuals=np.asarray(st.residuals),
                        dtau=np.asarray(st.dtau), seconds=dt)
    print(f"C4 (reduced): {disc.n_mac} macros, {disc.n_trace} trace dofs; newton {st.iterations}, "
          f"krylov {st.krylov_iterations}, residuals {np.array2string(np.asarray(st.residuals), precision=4)}, "
          f"dtau {np.array2string(np.asarray(st.dtau), precision=3)} in {dt:.1f} s")


if __name__ == "__main__":
    main()
