"""A/B: Schur-complement kernel variants (0 DMMA, 1 row blocks, 2 per-macro FFMA) on C2:
time of mhdg_schur_matrix and max relative difference of S against variant 2."""
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
ref = None
for v in [int(a) for a in sys.argv[1:]] or [2, 1, 0]:
    L.mhdg_set_schur_variant(v)
    S = cond.schur_matrix_into_factors()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        cond.schur_matrix_into_factors()
    e1.record()
    torch.cuda.synchronize()
    if ref is None:
        ref = S[:256].clone()
    err = float((S[:256] - ref).abs().max() / ref.abs().max())
    print(f"schur variant {v}: {e0.elapsed_time(e1) / 3:.2f} ms, rel diff vs first {err:.2e}", flush=True)
L.mhdg_set_schur_variant(0)
