"""A/B: split apply (pre / S^-1 stream / post) vs fused streamed kernel on C2."""
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
cond = CondensedSchur.build(blocks)
xs = torch.randn(22, disc.n_trace, dtype=torch.float64, device="cuda")
b = bench.algorithmic_bytes_per_macro(disc) * disc.n_mac
ys = {}
for split in (1, 0, 1, 0):
    L.mhdg_set_apply_split(split)
    ys[split] = cond.apply_trace(xs[0]).clone()
    for i in range(2):
        cond.apply_trace(xs[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20):
        cond.apply_trace(xs[2 + i])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"split={split}: {ms:.3f} ms/apply  {b / ms / 1e6:.0f} GB/s algorithmic")
print("split vs fused rel diff", float((ys[1] - ys[0]).abs().max() / ys[0].abs().max()))
