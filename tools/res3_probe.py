"""3D residual-only assembly on a TGV mesh (n1d^3 x 6 macros, m = 2, p = 2): workload for an ncu
capture of k_assemble<3> with want_jac = 0."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 8
c3 = TgvCase(reynolds=1600.0, mach=0.1)
d3 = Discretization(build_cube_mesh(c3.domain, n1d, 2, periodic=(True, True, True)), 2, c3.params)
u3, uh3 = d3.nodal_interpolant(c3.initial_state)
f = A.FieldState(torch.as_tensor(u3, device="cuda"), None, torch.as_tensor(uh3, device="cuda"))
f.q = A.gradient_refresh(d3, f.u, f.uhat)
ctx = A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02)
for _ in range(3):
    with _lib.Timeline(16) as tl:
        r = A.residual(d3, f, ctx)
        torch.cuda.synchronize()
    print(f"{d3.n_mac} macros: residual-only assemble kernel {tl.ms.get('assemble', 0):.3f} ms", flush=True)
