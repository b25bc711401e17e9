"""Cycle accounting of k_gj2 phases (tools/prof/libmhdg_prof.so, -DMHDG_STREAM_PROFILE)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib  # noqa: E402

_lib.LIB_PATH = os.path.join(ROOT, "tools", "prof", "libmhdg_prof.so")
import bench  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402

L = _lib.lib()
L.mhdg_gj_profile.argtypes = [C.c_void_p, C.c_int]
case, disc = bench.c2_discretization()
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
cond = CondensedSchur.build(blocks)
torch.cuda.synchronize()
L.mhdg_gj_profile(None, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
cond.refactor()
e1.record()
torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)()
L.mhdg_gj_profile(buf, 0)
a = np.array(buf, dtype=np.float64) / disc.n_mac
print(f"condense {e0.elapsed_time(e1):.1f} ms; cycles per macro (thread 0):")
for nm, v in zip(["panel load", "subpanel GJ steps", "subpanel DMMA", "row swaps", "big update", "write back", "  (LU: stage+U12)", "  (LU: trailing)"], a):
    print(f"  {nm:18s} {v:10.0f}")
