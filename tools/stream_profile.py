"""Cycle accounting of the streamed apply kernel (needs tools/prof/libmhdg_prof.so,
built with -DMHDG_STREAM_PROFILE).  Prints wait/compute/transition cycles per
piece kind summed over CTAs (thread 0 of each CTA)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "tools", "prof", "libmhdg_prof.so")
import bench  # noqa: E402
import torch  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402

L = _lib.lib()
L.mhdg_stream_profile.argtypes = [C.c_void_p, C.c_int]
if len(sys.argv) > 1 and sys.argv[1] == "c3":  # 3D TGV, 16^3 x 6 macros, m=2, p=2
    from paper_2402_11361_b200.cases import TgvCase
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.mesh import build_cube_mesh

    case = TgvCase(reynolds=1600.0, mach=0.1)
    disc = Discretization(build_cube_mesh(case.domain, 16, 2, periodic=(True, True, True)), 2, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    ctx = A.StageContext(50.0, torch.zeros((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device="cuda"),
                         float("inf"), 0.02)
else:
    case, disc = bench.c2_discretization()
    u, uhat = bench.c2_state(case, disc)
    ctx = A.StageContext.steady(1.0)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, ctx)
cond = CondensedSchur.build(blocks)
x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda")
cond.apply_trace(x)
torch.cuda.synchronize()
L.mhdg_stream_profile(None, 1)
reps = 5
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    cond.apply_trace(x)
e1.record()
torch.cuda.synchronize()
buf = (C.c_ulonglong * 48)()
L.mhdg_stream_profile(buf, 0)
a = np.array(buf, dtype=np.float64).reshape(16, 3)
names = ["FST", "FTT", "WV", "WFZ", "SI", "Y2", "FC", "-", "WF2", "FTS", "GF", "MD", "END", "MSTART", "Y1", "WB"]
ms = e0.elapsed_time(e1) / reps
L.mhdg_stream_grid.restype = C.c_int
ncta = L.mhdg_stream_grid()
print("grid", ncta)
tot = a.sum()
print(f"apply {ms:.3f} ms; per-CTA cycles/apply {tot / reps / ncta:.0f} (clock ~1.965 GHz -> {ms * 1.965e6:.0f})")
for i, nm in enumerate(names):
    w, c, t = a[i] / reps / ncta
    if w + c + t > 0:
        print(f"{nm:4s} wait {w:9.0f}  compute {c:9.0f}  transition {t:9.0f}")
