"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): every library kernel family once on a 3D TGV m=2, p=2 cube (6
macros, the streamed split apply with its mbarrier/bulk-copy ring, the packed
LU, the preconditioner, rhs/recover, the ICGS) and on a 2D C2-shape (m=4, p=3)
periodic patch.  Prints one line per case; exits non-zero on a parity miss.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import krylov as K  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase, UniformFlow2D  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh, build_square_mesh  # noqa: E402


def run(name, disc, u, uhat, ctx):
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    res = A.residual(disc, f, ctx)
    blocks, _ = A.jacobian(disc, f, ctx)
    cond = CondensedSchur.build(blocks)
    x = torch.as_tensor(np.random.default_rng(1).standard_normal(disc.n_trace), device="cuda")
    y = cond.apply_trace(x)
    b = cond.rhs(*res)
    du, dq = cond.recover(res[0], res[1], x)
    r, nmv = K.solve_trace_system(cond, b, K.KrylovConfig(rel_tol=1e-6, max_iter=30, restart=10, inner_iter=3),
                                  "fgmres")
    cond.form_local_operators()
    y2 = cond.apply_trace(x)
    err = float((y2 - y).abs().max() / y.abs().max())
    torch.cuda.synchronize()
    print(f"{name}: {disc.n_mac} macros, |y| {float(y.norm()):.3e}, stored-vs-matrix-free {err:.1e}, "
          f"fgmres {r.iterations} its, {nmv} matvecs, |du| {float(du.norm()):.3e}", flush=True)
    return err < 1e-9


def main():
    torch.cuda.set_device(0)
    ok = True
    tgv = TgvCase(reynolds=1600.0, mach=0.1)
    d3 = Discretization(build_cube_mesh(tgv.domain, 1, 2, periodic=(True,) * 3), 2, tgv.params)
    u, uh = d3.nodal_interpolant(tgv.initial_state)
    ctx = A.StageContext(50.0, torch.as_tensor(-0.3 * u, device="cuda"), np.inf, 0.02)
    ok &= run("3D TGV m2p2", d3, u, uh, ctx)
    c2 = UniformFlow2D()
    d2 = Discretization(build_square_mesh(c2.domain, 2, 4, periodic=(True, True)), 3, c2.params)
    u, uh = d2.nodal_interpolant(c2.state)
    ok &= run("2D C2-shape m4p3", d2, u, uh, A.StageContext.steady(1.0))
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
