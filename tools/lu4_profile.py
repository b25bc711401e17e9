"""Cycle accounting of k_lu4 phases on C2 (tools/prof/libmhdg_prof.so, -DMHDG_STREAM_PROFILE);
thread 0 of every CTA, summed, per macro."""
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
from paper_2402_11361_b200 import condense as CD  # noqa: E402

CD.FACTOR = "lu"
L = _lib.lib()
L.mhdg_lu4_profile.argtypes = [C.c_void_p, C.c_int]
case, disc = bench.c2_discretization(int(sys.argv[1]) if len(sys.argv) > 1 else 64)
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
cond = CD.CondensedSchur.build(blocks)
torch.cuda.synchronize()
L.mhdg_lu4_profile(None, 1)
with _lib.Timeline(64) as tl:
    cond.refactor()
    torch.cuda.synchronize()
buf = (C.c_ulonglong * 8)()
L.mhdg_lu4_profile(buf, 0)
a = np.array(buf, dtype=np.float64) / disc.n_mac
print("kernels:", ", ".join(f"{k} {v:.2f} ms" for k, v in tl.ms.items()))
print("cycles per macro (thread 0):")
for nm, v in zip(["panel load", "sub-panel pivot steps", "(a)+(b) intra-panel", "write/compact/inv(L11)",
                  "trailing (warp 0's chunks)", "trailing barrier wait"], a):
    print(f"  {nm:28s} {v:10.0f}")
print(f"  {'total':28s} {a[:6].sum():10.0f}")
