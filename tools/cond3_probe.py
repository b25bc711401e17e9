"""3D condensation on a TGV mesh (n1d^3 x 6 macros, m = 2, p = 2): workload for ncu captures of
k_schur2 / k_lu4 (sh tools/prof_kernel.sh TAG k_schur2 1 -- python tools/cond3_probe.py 12)."""
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

n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 12
case = TgvCase(reynolds=1600.0, mach=0.1)
disc = Discretization(build_cube_mesh(case.domain, n1d, 2, periodic=(True,) * 3), 2, case.params)
u, uhat = disc.nodal_interpolant(case.initial_state)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
ctx = A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02)
blocks, _ = A.jacobian(disc, f, ctx)
cond = CondensedSchur.allocate(blocks)
st = disc.device.status_buffer()
for _ in range(3):
    with _lib.Timeline(16) as tl:
        cond.refactor_async(st)
        torch.cuda.synchronize()
    print(disc.n_mac, {k: round(v, 3) for k, v in tl.ms.items()}, flush=True)
A.raise_status(st, "condense")
