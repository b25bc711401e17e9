"""Short driver for ncu captures of the condensation and apply kernels at a BASELINE
size: one Jacobian, two condensations (Schur, LU, pack), one split apply.

    python tools/prof_ops.py C3|C2
    ncu --set full --clock-control none --import-source on \
        -k regex:"k_schur2|k_lu4|k_pack_lu4|k_apply_stream" -s 3 -c 5 -o OUT python tools/prof_ops.py C3
(-s 3 skips the first condensation's kernels; the capture is the second condensation
and the apply's pre and post kernels.)
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402


def main(cfg):
    torch.cuda.set_device(0)
    if cfg == "C2":
        case, disc = bench.c2_discretization()
        u, uhat = bench.c2_state(case, disc)
        ctx = A.StageContext.steady(1.0)
        hist = None
    else:
        case = TgvCase(reynolds=1600.0, mach=0.1)
        disc = Discretization(build_cube_mesh(case.domain, 16, 2, periodic=(True,) * 3), 2, case.params)
        u, uhat = disc.nodal_interpolant(case.initial_state)
        hist = torch.zeros((disc.n_mac, disc.L, disc.ns), dtype=torch.float64, device="cuda")
        ctx = A.StageContext(50.0, hist, np.inf, 0.02)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    blocks, _ = A.jacobian(disc, f, ctx)
    cond = CondensedSchur.allocate(blocks)
    st = disc.device.status_buffer()
    cond.refactor_async(st)
    cond.refactor_async(st)
    x = torch.as_tensor(np.random.default_rng(1).standard_normal(disc.n_trace), device="cuda")
    y = cond.apply_trace(x)
    torch.cuda.synchronize()
    A.raise_status(st, "condense")
    print(cfg, "ok", float(y.norm()))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3")
