"""A/B of the streamed apply's L2 prefetch lookahead at C3 (3D TGV, 24,576 macros):
split-apply time and per-kernel times (library timeline), 20 applies per setting.

    python tools/ab_c3_apply.py [lookaheads...]
"""
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

case = TgvCase(reynolds=1600.0, mach=0.1)
disc = Discretization(build_cube_mesh(case.domain, 16, 2, periodic=(True,) * 3), 2, case.params)
u, uhat = disc.nodal_interpolant(case.initial_state)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
ctx = A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02)
blocks, _ = A.jacobian(disc, f, ctx)
cond = CondensedSchur.build(blocks)
L = _lib.lib()
xs = torch.as_tensor(np.random.default_rng(1).standard_normal((4, disc.n_trace)), device="cuda")
y = torch.empty(disc.n_trace, dtype=torch.float64, device="cuda")
bref = bench.algorithmic_bytes_per_macro(disc) * disc.n_mac
hbm = float(bench.measured_peaks().get("hbm_gbs", 6550.0))
for pa in [int(a) for a in sys.argv[1:]] or [0, 2, 3, 4, 6, 8, 12]:
    L.mhdg_set_stream_prefetch(pa)
    for i in range(3):
        cond.apply_trace(xs[i & 3], out=y)
    torch.cuda.synchronize()
    K = 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with _lib.Timeline(8 * K + 8) as tl:
        e0.record()
        for i in range(K):
            cond.apply_trace(xs[i & 3], out=y)
        e1.record()
        e1.synchronize()
    t = e0.elapsed_time(e1) / K
    ks = {k: round(tl.ms[k] / tl.counts[k], 3) for k in tl.ms}
    print(f"prefetch {pa:2d}: apply {t:.3f} ms = {bref / t / 1e6 / hbm:.3f} of B_ref roofline; {ks}", flush=True)
L.mhdg_set_stream_prefetch(-1)
