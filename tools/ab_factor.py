"""A/B: Gauss-Jordan factor variants (2: row interchanges, 3: pivots in place) on C2;
times the full condensation (Schur + inverse + tiling) and compares the inverses."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402

L = _lib.lib()
case, disc = bench.c2_discretization()
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
cond = CondensedSchur.allocate(blocks)
st = disc.device.status_buffer()
inv = {}
for v in [int(a) for a in sys.argv[1:]] or [2, 3, 2, 3]:
    L.mhdg_set_factor_variant(v)
    cond.refactor_async(st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        cond.refactor_async(st)
    e1.record()
    torch.cuda.synchronize()
    A.raise_status(st, "condense")
    inv[v] = cond.lu.clone()
    print(f"variant {v}: {e0.elapsed_time(e1) / 3:.2f} ms per condensation", flush=True)
if 2 in inv and 3 in inv:
    print("inverse rel diff", float((inv[3] - inv[2]).abs().max() / inv[2].abs().max()))
L.mhdg_set_factor_variant(3)
