"""A/B: factor kinds on C2 (explicit inverse by Gauss-Jordan vs packed LU):
condensation time and agreement of apply / rhs / recover."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import condense as CD  # noqa: E402

n_cells = int(sys.argv[1]) if len(sys.argv) > 1 else 64
case, disc = bench.c2_discretization(n_cells)
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
ctx = A.StageContext.steady(1.0)
res = A.residual(disc, f, ctx)
blocks, _ = A.jacobian(disc, f, ctx)
x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda")
out = {}
for kind in ("inverse", "lu"):
    CD.FACTOR = kind
    cond = CD.CondensedSchur.allocate(blocks)
    st = disc.device.status_buffer()
    cond.refactor_async(st)
    torch.cuda.synchronize()
    A.raise_status(st, "condense")
    with _lib.Timeline(64) as tl:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(2):
            cond.refactor_async(st)
        e1.record()
        torch.cuda.synchronize()
    A.raise_status(st, "condense")
    y = cond.apply_trace(x)
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record()
    for _ in range(5):
        cond.apply_trace(x)
    eb.record()
    torch.cuda.synchronize()
    b = cond.rhs(*res)
    du, dq = cond.recover(res[0], res[1], x)
    out[kind] = (y.clone(), b.clone(), du.clone())
    print(f"{kind:8s}: condense {e0.elapsed_time(e1) / 2:.2f} ms  kernels "
          + ", ".join(f"{k} {v / 2:.2f}" for k, v in tl.ms.items()) + f"; apply {ea.elapsed_time(eb) / 5:.3f} ms", flush=True)
CD.FACTOR = "inverse"
for i, name in enumerate(("apply", "rhs", "recover du")):
    a, c = out["inverse"][i], out["lu"][i]
    print(f"{name}: lu vs inverse rel diff {float((a - c).abs().max() / c.abs().max()):.2e}")
