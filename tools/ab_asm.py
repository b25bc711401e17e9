"""A/B: assembly kernel time (Jacobian + residual) on C2 and C3."""
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
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

case, disc = bench.c2_discretization(64)
u, uhat = bench.c2_state(case, disc)
c3 = TgvCase(reynolds=1600.0, mach=0.1)
d3 = Discretization(build_cube_mesh(c3.domain, 16, 2, periodic=(True, True, True)), 2, c3.params)
u3, uh3 = d3.nodal_interpolant(c3.initial_state)
for name, d, uu, uh, ctx in (("C2", disc, u, uhat, A.StageContext.steady(1.0)),
                             ("C3", d3, u3, uh3, A.StageContext(50.0, None, np.inf, 0.02))):
    f = A.FieldState(torch.as_tensor(uu, device="cuda"), None, torch.as_tensor(uh, device="cuda"))
    f.q = A.gradient_refresh(d, f.u, f.uhat)
    if ctx.hist is None and ctx.dt_coeff != 0.0:
        ctx.hist = torch.zeros_like(f.u)
    blocks, _ = A.jacobian(d, f, ctx)
    del blocks
    torch.cuda.synchronize()
    with _lib.Timeline(16) as tl:
        blocks, _ = A.jacobian(d, f, ctx)
        torch.cuda.synchronize()
    print(f"{name}: assemble kernel {tl.ms.get('assemble', 0):.2f} ms", flush=True)
    del blocks, f
    torch.cuda.empty_cache()
