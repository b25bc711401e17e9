"""A/B: chunk-pipelined split apply (mhdg_set_apply_pipeline) vs the sequential split
apply at C2 (or C3): apply time over 20 applies (CUDA events on the caller's stream),
bitwise equality of the result.

    python tools/ab_pipeline.py C2|C3
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
cond = CondensedSchur.build(blocks)
L = _lib.lib()
xs = torch.as_tensor(np.random.default_rng(1).standard_normal((4, disc.n_trace)), device="cuda")
y = torch.empty(disc.n_trace, dtype=torch.float64, device="cuda")
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def timed(k=20):
    for i in range(3):
        cond.apply_trace(xs[i & 3], out=y)
    torch.cuda.synchronize()
    a, b = ev(), ev()
    a.record()
    for i in range(k):
        cond.apply_trace(xs[i & 3], out=y)
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / k


L.mhdg_set_apply_pipeline(0, 0, 0, 0)
y_ref = cond.apply_trace(xs[0]).clone()
base = timed()
print(f"{cfg} sequential: {base:.4f} ms", flush=True)
sms = 148
for chunks in (2, 4, 8, 16):
    for cp, cs, cq in ((sms, 0, sms), (sms, 4 * sms, sms), (sms, 8 * sms, sms), (0, 0, 0), (2 * sms, 0, sms)):
        L.mhdg_set_apply_pipeline(chunks, cp, cs, cq)
        t = timed()
        same = bool(torch.equal(cond.apply_trace(xs[0]), y_ref))
        print(f"{cfg} chunks {chunks:2d} caps pre {cp} solve {cs} post {cq}: {t:.4f} ms ({base / t:.3f}x)  "
              f"bitwise {same}", flush=True)
L.mhdg_set_apply_pipeline(0, 0, 0, 0)
