"""C1 golden fixture from the oracle (test infrastructure; parity of the 2D
path rests on the oracle, itself pinned to the reference in 3D by
tests/test_oracle_golden.py).

BASELINE configs[0]: [0,2]x[0,1], 8x4 squares split SW->NE (64 macros), m=2,
p=2, gamma=1.4, Pr=0.72, Re=100, M=0.15, acoustic scaling (wall speed
M c_inf, T_wall=1 on both walls), x-periodic.  IC: exact plane Couette at the
nodes and owner-side traces plus U(-1e-3, 1e-3) on every U and U-hat
coefficient (default_rng(0)), q = gradient_refresh.  PTC + FGMRES to
relative residual 1e-10.  Writes tests/golden/c1_ptc_oracle.npz (the
reference's explicit-inverse Schur factors, condense.py:67) or, with ``lu``,
tests/golden/c1_ptc_oracle_lu.npz (LAPACK LU solves: the algebra of the
device's default packed-LU factors).  Both record the accepted state after
every Newton step and the per-step FGMRES counts.

    python oracle/make_c1_golden.py [inv|lu]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle.hdg_oracle as O  # noqa: E402
from paper_2402_11361_b200.cases import CouettePlane2D  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_square_mesh  # noqa: E402


def c1_setup():
    case = CouettePlane2D()
    mesh = build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False))
    disc = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
    u, uhat = disc.nodal_interpolant(case.exact_state)
    rng = np.random.default_rng(0)
    u = u + rng.uniform(-1e-3, 1e-3, u.shape)
    uhat = uhat + rng.uniform(-1e-3, 1e-3, uhat.shape)
    return case, disc, u, uhat


def main(mode="inv"):
    case, disc, u, uhat = c1_setup()
    q = O.gradient_refresh(disc, u, uhat)
    f = O.Fields(u.copy(), q.copy(), uhat.copy())
    steps_u, steps_uhat = [], []

    def log(st, fields):
        steps_u.append(fields.u.copy())
        steps_uhat.append(fields.uhat.copy())
        print(f"  newton {st.iterations}: residual {st.residuals[-1]:.4e}, fgmres {st.krylov_per_step[-1]}",
              flush=True)

    t0 = time.perf_counter()
    st, _ = O.ptc_steady_solve(disc, f, rel_tol=1e-10, log=log, mode=mode)
    dt = time.perf_counter() - t0
    name = "c1_ptc_oracle.npz" if mode == "inv" else f"c1_ptc_oracle_{mode}.npz"
    out = os.path.join(ROOT, "tests", "golden", name)
    np.savez_compressed(out, u0=u, q0=q, uhat0=uhat, u=f.u, q=f.q, uhat=f.uhat, newton=st.iterations,
                        krylov=st.krylov_iterations, residuals=np.asarray(st.residuals), seconds=dt,
                        krylov_per_step=np.asarray(st.krylov_per_step), dtau=np.asarray(st.dtau),
                        steps_u=np.stack(steps_u), steps_uhat=np.stack(steps_uhat), mode=mode)
    print(f"C1: {disc.n_mac} macros, {disc.n_trace} trace dofs; newton {st.iterations}, "
          f"krylov {st.krylov_iterations}, residuals {st.residuals[0]:.3e} -> {st.residuals[-1]:.3e} in {dt:.1f} s")


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "inv")
