"""A/B of the face-block preconditioner build: register-tile Gauss-Jordan sweep (default)
against the shared-memory Cholesky + triangular inverse, at C2 and C3 (and a few other
(d, m, p) for the tile sizes): time per build, agreement of the inverses, and the residual
||B inv - I|| of each against the symmetrised block it inverts."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.krylov import BlockPreconditioner  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

L = _lib.lib()


def run(name, disc, f, ctx):
    blocks, _ = A.jacobian(disc, f, ctx)
    cond = CondensedSchur.allocate(blocks)
    out = {}
    for var in (1, 0):
        L.mhdg_set_precond_variant(var)
        pre = BlockPreconditioner(cond)
        torch.cuda.synchronize()
        with _lib.Timeline(16) as tl:
            for _ in range(3):
                pre = BlockPreconditioner(cond)
            torch.cuda.synchronize()
        out[var] = (pre.inverse.clone(), tl.ms["precond_build"] / 3)
    L.mhdg_set_precond_variant(0)
    i1, t1 = out[1]
    i0, t0 = out[0]
    rel = float((i0 - i1).abs().max() / i1.abs().max())
    x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda")
    bs = disc.Lf * disc.ns
    y0 = torch.bmm(i0, x.view(-1, bs, 1)).view(-1)
    y1 = torch.bmm(i1, x.view(-1, bs, 1)).view(-1)
    rely = float((y0 - y1).abs().max() / y1.abs().max())
    asym = float((i0 - i0.transpose(1, 2)).abs().max() / i0.abs().max())
    print(f"{name}: faces {disc.mesh.n_faces}, bs {bs}: shared-memory Cholesky {t1:.3f} ms, register sweep {t0:.3f} ms "
          f"({t1 / t0:.1f}x); max rel diff of inverses {rel:.2e}, of inv x {rely:.2e}; asymmetry of the sweep's inverse {asym:.2e}",
          flush=True)


which = sys.argv[1:] or ["c2", "c3"]
if "c2" in which:
    case, disc = bench.c2_discretization()
    u, uhat = bench.c2_state(case, disc)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    run("C2", disc, f, A.StageContext.steady(1.0))
    del disc, f
for key, n1d, m, p in (("c3", 16, 2, 2), ("m1p1", 16, 1, 1), ("m1p2", 16, 1, 2), ("m1p3", 12, 1, 3), ("m2p3", 4, 2, 3)):
    if key not in which:
        continue
    case = TgvCase(reynolds=1600.0, mach=0.1)
    disc = Discretization(build_cube_mesh(case.domain, n1d, m, periodic=(True, True, True)), p, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    run(f"3D (m, p) = ({m}, {p})", disc, f, A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02))
    del disc, f
    torch.cuda.empty_cache()
