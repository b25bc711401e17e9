"""A/B: LU kernels (k_lu3 vs k_lu4) and the explicit inverse on C2 : factor time and agreement of the condensed apply."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import condense as CD  # noqa: E402

L = _lib.lib()
case, disc = bench.c2_discretization(int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 64)
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
out = {}
VARIANTS = (("inverse", "inverse", 0, 32, 0), ("lu3", "lu", 3, 32, 0), ("lu4", "lu", 4, 32, 0),
            ("lu4b", "lu", 4, 32, 0), ("lu4_64x256", "lu", 4, 64, 256), ("lu4_64x384", "lu", 4, 64, 384))
for label, kind, var, nb, nt in VARIANTS:
    CD.FACTOR = kind
    if var:
        L.mhdg_set_lu_variant(var)
        L.mhdg_set_lu_panel(nb, nt)
    cond = CD.CondensedSchur.allocate(blocks)
    st = disc.device.status_buffer()
    cond.refactor_async(st)
    torch.cuda.synchronize()
    A.raise_status(st, "condense")
    with _lib.Timeline(64) as tl:
        for _ in range(2):
            cond.refactor_async(st)
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
    out[label] = y.clone()
    print(f"{label:8s}: " + ", ".join(f"{k} {v / 2:.2f} ms" for k, v in tl.ms.items())
          + f"; apply {ea.elapsed_time(eb) / 5:.3f} ms", flush=True)
    del cond
CD.FACTOR = "inverse"
ref = out["inverse"]
for k, v in out.items():
    print(f"{k}: vs inverse rel diff {float((v - ref).abs().max() / ref.abs().max()):.2e}")
print("lu4 run-to-run equal:", bool(torch.equal(out["lu4"], out["lu4b"])))
L.mhdg_set_lu_panel(32, 0)
