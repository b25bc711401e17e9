"""A/B: k_lu4 with a persistent grid (fewer resident trailing matrices) x L2 policy,
at C2 and C3 (factor kernel time from the library timeline, median of 3).

    python tools/ab_lu_grid.py C2|C3
"""
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
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
if cfg == "C2":
    case, disc = bench.c2_discretization()
    u, uhat = bench.c2_state(case, disc)
    ctx = A.StageContext.steady(1.0)
else:
    case = TgvCase(reynolds=1600.0, mach=0.1)
    disc = Discretization(build_cube_mesh(case.domain, 16, 2, periodic=(True,) * 3), 2, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    ctx = A.StageContext(50.0, torch.zeros((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device="cuda"),
                         np.inf, 0.02)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, ctx)
cond = CondensedSchur.allocate(blocks)
st = disc.device.status_buffer()
L = _lib.lib()
x = torch.as_tensor(np.random.default_rng(1).standard_normal(disc.n_trace), device="cuda")
cond.refactor_async(st)
y_ref = cond.apply_trace(x).clone()
for grid in (0, 148, 185, 222, 259, 296):
    for l2 in (2, 0):
        L.mhdg_set_lu_grid(grid)
        L.mhdg_set_lu_l2mode(l2)
        ts = []
        for _ in range(3):
            with _lib.Timeline(64) as tl:
                cond.refactor_async(st)
                torch.cuda.synchronize()
            ts.append(tl.ms["factor"])
        y = cond.apply_trace(x)
        same = bool(torch.equal(y, y_ref))
        print(f"{cfg} grid {grid:4d} l2mode {l2}: factor {np.median(ts):.3f} ms  (apply bitwise same: {same})",
              flush=True)
L.mhdg_set_lu_grid(0)
L.mhdg_set_lu_l2mode(2)
