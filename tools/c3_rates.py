"""C3 (3D TGV, 16^3 x 6 macros, m=2, p=2) rates: apply (split / fused / generic),
condensation, assembly -- for DESIGN's table (not a bench line)."""
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

n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
case = TgvCase(reynolds=1600.0, mach=0.1)
disc = Discretization(build_cube_mesh(case.domain, n1d, 2, periodic=(True, True, True)), 2, case.params)
u, uhat = disc.nodal_interpolant(case.initial_state)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
ctx = A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02)
L = _lib.lib()
if os.environ.get("MHDG_PREF"):  # A/B: L2 prefetch lookahead of the streamed kernels (pieces)
    L.mhdg_set_stream_prefetch(int(os.environ["MHDG_PREF"]))
blocks, _ = A.jacobian(disc, f, ctx)
del blocks
torch.cuda.synchronize()
with _lib.Timeline(16) as ta:
    blocks, _ = A.jacobian(disc, f, ctx)
    torch.cuda.synchronize()
cond = CondensedSchur.allocate(blocks)
st = disc.device.status_buffer()
cond.refactor_async(st)
torch.cuda.synchronize()
with _lib.Timeline(16) as tc:
    cond.refactor_async(st)
    torch.cuda.synchronize()
A.raise_status(st, "condense")
x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda")
b_mac = bench.algorithmic_bytes_per_macro(disc)
HBM = float(bench.measured_peaks().get("hbm_gbs", 6533.2))  # GB/s, as bench.py
print(f"C3: {disc.n_mac} macros, n_trace {disc.n_trace}, B_ref {b_mac / 1e3:.1f} KB/macro, "
      f"{b_mac * disc.n_mac / 1e9:.2f} GB/apply")
print(f"assembly kernel {ta.ms.get('assemble', 0):.2f} ms = {disc.n_mac / ta.ms.get('assemble', 1) * 1e3:.3g} macros/s")
tot = sum(tc.ms.values())
print(f"condense {tot:.2f} ms = {disc.n_mac / tot * 1e3:.3g} macros/s  " + ", ".join(f"{k} {v:.2f}" for k, v in tc.ms.items()))
for name, split, stream in (("split", 1, 1), ("fused", 0, 1), ("generic", 1, 0)):
    L.mhdg_set_apply_split(split)
    L.mhdg_set_stream_enabled(stream)
    for _ in range(2):
        cond.apply_trace(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        cond.apply_trace(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"apply {name:8s} {ms:.3f} ms = {disc.n_trace / ms * 1e3:.3g} DOF-applies/s, "
          f"{b_mac * disc.n_mac / ms / 1e6:.0f} GB/s (B_ref) = {b_mac * disc.n_mac / ms / 1e6 / HBM:.3f}")
L.mhdg_set_apply_split(1)
L.mhdg_set_stream_enabled(1)
kb = bench.apply_kernel_bytes(disc)
with _lib.Timeline(256) as tl:
    for _ in range(10):
        cond.apply_trace(x)
    torch.cuda.synchronize()
for k, v in tl.ms.items():
    ms = v / tl.counts[k]
    extra = f", {kb[k] / ms / 1e6:.0f} GB/s = {kb[k] / ms / 1e6 / HBM:.2f}" if k in kb else ""
    print(f"  {k:12s} {ms:.3f} ms{extra}")

# stored local operators (B_A): formation time, apply rate, agreement with the matrix-free apply
if os.environ.get("MHDG_C3_STORED", "1") != "0":
    y_mf = cond.apply_trace(x).clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    at = cond.form_local_operators()
    e1.record()
    torch.cuda.synchronize()
    t_form = e0.elapsed_time(e1)
    ltr = disc.nf * disc.Lf * disc.ns
    b_st = (8 * ltr * ltr + 12 * ltr) * disc.n_mac
    for _ in range(2):
        y_st = cond.apply_trace(x)
    torch.cuda.synchronize()
    rel = float((y_st - y_mf).abs().max() / y_mf.abs().max())
    e0.record()
    for _ in range(10):
        cond.apply_trace(x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"apply stored   {ms:.3f} ms = {disc.n_trace / ms * 1e3:.3g} DOF-applies/s, {b_st / ms / 1e6:.0f} GB/s "
          f"(B_A {b_st / disc.n_mac / 1e3:.1f} KB/macro) = {b_st / ms / 1e6 / HBM:.3f}; formation {t_form:.1f} ms; "
          f"max rel diff vs matrix-free {rel:.2e}")
