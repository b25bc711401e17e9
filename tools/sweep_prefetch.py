"""Time the C2 apply for several L2-prefetch lookaheads of the streamed kernel."""
import ctypes as C
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
L.mhdg_set_stream_prefetch.argtypes = [C.c_int]
case, disc = bench.c2_discretization()
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
cond = CondensedSchur.build(blocks)
xs = torch.randn(12, disc.n_trace, dtype=torch.float64, device="cuda")
b = bench.algorithmic_bytes_per_macro(disc) * disc.n_mac
for pa in [int(a) for a in sys.argv[1:]] or [0, 2, 4, 8, 16]:
    L.mhdg_set_stream_prefetch(pa)
    for i in range(2):
        cond.apply_trace(xs[i])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(10):
        cond.apply_trace(xs[2 + i])
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"prefetch {pa:3d}: {ms:.3f} ms/apply  {b / ms / 1e6:.0f} GB/s algorithmic")
