"""Coupling-recompute representation (B_min) at C3 size (3D TGV, n^3 x 6 macros, m=2,
p=2): build time, apply time per window size, resident device memory against the
resident-blocks representation, and bitwise agreement of the two applies.

    python tools/recompute_rates.py [n_ele_1d=16] [chunks=1024,4096,8192]
"""
import json
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
from paper_2402_11361_b200.condense import CondensedSchur, condense  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402

n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
chunks = [int(c) for c in (sys.argv[2] if len(sys.argv) > 2 else "1024,4096,8192").split(",")]
resident = os.environ.get("MHDG_RESIDENT", "1") != "0"  # 0: skip the resident reference (it may not fit)
case = TgvCase(reynolds=1600.0, mach=0.1)
disc = Discretization(build_cube_mesh(case.domain, n1d, 2, periodic=(True, True, True)), 2, case.params)
f = A.interpolate(disc, case.initial_state)
ctx = A.StageContext(50.0, torch.zeros_like(f.u), np.inf, 0.02)
x = torch.randn(disc.n_trace, dtype=torch.float64, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1))
HBM = float(bench.measured_peaks().get("hbm_gbs", 6533.2))
b_ref = bench.algorithmic_bytes_per_macro(disc)
n, ltr = disc.L * disc.ns, disc.nf * disc.Lf * disc.ns
b_min = 8 * (n * n + 3 * ltr + n + (1 + 9 + 12 + 8)) + 4 * ltr


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"n_macros": disc.n_mac, "n_trace": disc.n_trace, "B_ref_KB": b_ref / 1e3, "B_min_KB": b_min / 1e3}
base = torch.cuda.memory_allocated()
y_ref = None
if resident:
    torch.cuda.reset_peak_memory_stats()
    blocks, fro = A.jacobian(disc, f, ctx, recompute=False)
    cond0 = CondensedSchur.build(blocks)
    pre0 = A and __import__("paper_2402_11361_b200.krylov", fromlist=["x"]).block_precond_build(cond0)
    torch.cuda.synchronize()
    out["resident"] = {"device_GB": (torch.cuda.memory_allocated() - base) / 1e9,
                       "peak_GB": (torch.cuda.max_memory_allocated() - base) / 1e9,
                       "apply_ms": timed(lambda: cond0.apply_trace(x), 10)}
    y_ref = cond0.apply_trace(x).clone()
    lu_ref = cond0.lu.clone() if disc.n_mac <= 30000 else None
    del blocks, fro, cond0, pre0
    torch.cuda.empty_cache()
out["recompute"] = []
for c in chunks:
    torch.cuda.reset_peak_memory_stats()
    m0 = torch.cuda.memory_allocated()
    rb = A.RecomputeBlocks(disc, f, ctx, chunk=c)
    cond = condense(rb)
    torch.cuda.synchronize()
    t_build = timed(cond.refactor, 2)
    with _lib.Timeline(4096) as tl:
        cond.apply_trace(x)
        torch.cuda.synchronize()
    t_apply = timed(lambda: cond.apply_trace(x), 5)
    rec = {"chunk": rb.chunk, "build_ms": t_build, "apply_ms": t_apply,
           "apply_kernels_ms": {k: v for k, v in tl.ms.items()},
           "device_GB": (torch.cuda.memory_allocated() - m0) / 1e9,
           "peak_GB": (torch.cuda.max_memory_allocated() - m0) / 1e9,
           "dof_applies_per_s": disc.n_trace / t_apply * 1e3,
           "B_min_GBs": b_min * disc.n_mac / t_apply / 1e6}
    if y_ref is not None:
        rec["apply_bitwise_equal_resident"] = bool(torch.equal(cond.apply_trace(x), y_ref))
        if lu_ref is not None:
            rec["factors_bitwise_equal_resident"] = bool(torch.equal(cond.lu, lu_ref))
    out["recompute"].append(rec)
    print(json.dumps(rec), flush=True)
    del cond, rb
    torch.cuda.empty_cache()
print(json.dumps(out))
