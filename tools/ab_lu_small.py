"""A/B: the 96-thread / four-CTAs-per-SM LU (n <= 192) against the 192-thread kernel, on
C3 (n = 175) and C5-shaped TGV meshes ((1,2): n = 50, (1,3): n = 100), factor kernel time
from the library timeline (median of 3) and bitwise equality of the resulting apply.

    python tools/ab_lu_small.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

L = _lib.lib()
case = TgvCase(reynolds=1600.0, mach=0.1)
for n1d, m, p in ((16, 2, 2), (24, 1, 2), (20, 1, 3), (32, 1, 1), (24, 2, 1)):
    disc = Discretization(build_cube_mesh(case.domain, n1d, m, periodic=(True,) * 3), p, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    ctx = A.StageContext(50.0, torch.zeros((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device="cuda"),
                         np.inf, 0.02)
    blocks, _ = A.jacobian(disc, f, ctx)
    cond = CondensedSchur.allocate(blocks)
    st = disc.device.status_buffer()
    x = torch.as_tensor(np.random.default_rng(1).standard_normal(disc.n_trace), device="cuda")
    ys = {}
    for small in (0, 1, 2):
        L.mhdg_set_lu_small(small)
        cond.refactor_async(st)
        ts = []
        for _ in range(3):
            with _lib.Timeline(64) as tl:
                cond.refactor_async(st)
                torch.cuda.synchronize()
            ts.append(tl.ms["factor"])
        A.raise_status(st, "condense")
        ys[small] = cond.apply_trace(x).clone()
        print(f"(m,p)=({m},{p}) n={disc.L * disc.ns} macros={disc.n_mac} small={small}: factor {np.median(ts):.3f} ms",
              flush=True)
    print("  apply bitwise same:", bool(torch.equal(ys[0], ys[1])), bool(torch.equal(ys[0], ys[2])),
          "rel diff %.2e" % float((ys[0] - ys[1]).abs().max() / ys[0].abs().max()), flush=True)
    del cond, blocks
    torch.cuda.empty_cache()
L.mhdg_set_lu_small(1)
