"""C5 (BASELINE configs[4]) on one B200: Taylor-Green on 32^3 hexes x 6 Kuhn tets
(196,608 macros), macro subdivision m in {1, 2, 4} x p in {1, 2, 3}.  Per (m, p):
one Jacobian at the DIRK33 stage-1 context (dt = 0.01), its condensation (Schur +
batched LU, timed), then 200 trace-operator applies on x ~ N(0, 1) (seed 1, timed).

Combos whose device data exceed one GPU run the rank-0 slab of a P-GPU contiguous
slab partition (the macros this GPU would own with P = 2, 4, 8 GPUs; partition.py),
the smallest P that fits; "n_gpus_needed" says which.  The Schur scratch is bounded
to CHUNK macros (condensed chunk by chunk, mhdg_factors.scratch_macros) so the
resident data are the blocks plus the packed factors.  Combos beyond 8 GPUs or the
factor kernels' limit (mhdg_factor_max_n) are listed as such.

    python tools/c5_sweep.py [n_ele_1d]   (default 32)     -> one JSON line per combo
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import stepper as S  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.condense import CondensedRecompute, CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402
from paper_2402_11361_b200.partition import partition_mesh  # noqa: E402
from paper_2402_11361_b200.refmacro import lattice_size  # noqa: E402

N1D = int(sys.argv[1]) if len(sys.argv) > 1 else 32
BUDGET = 160e9  # bytes of device data per GPU (of ~180 GB HBM3e)
CHUNK = 4096  # macros of Schur scratch
# MHDG_C5_REPR=recompute: the coupling-recompute representation (B_min: only the S factors
# resident, the couplings re-formed per window of CHUNK macros before each local apply)
REPR = os.environ.get("MHDG_C5_REPR", "matrix_free")
L_ = _lib.lib()


def bytes_per_macro(m, p):
    """Device bytes per macro: blocks (state_state, 3 face blocks, stashes), the Schur
    scratch and its packed factor, the apply work area, fields/residuals (3D)."""
    d, ns, nf = 3, 5, 4
    L, Lf = lattice_size(d, m * p), lattice_size(d - 1, m * p)
    nq, nqf = (p + 1) ** d, (p + 1) ** (d - 1)
    n = L * ns
    blk = n * n + 3 * nf * (Lf * ns) ** 2 + m**d * nq * d * d * ns * ns + nf * m ** (d - 1) * nqf * d * ns * ns
    if REPR == "recompute":  # the factor and the vectors; the blocks exist for CHUNK macros only
        return 8 * (1.1 * n * n + 8 * n + 30 * L * ns) + 8.0 * (blk + 3 * n * n) * CHUNK / (6 * N1D**3)
    return 8 * (blk + 1.1 * n * n + 8 * n + 20 * L * ns)  # + the packed factor (scratch: CHUNK macros)


def run(m, p):
    n = lattice_size(3, m * p) * 5
    out = {"m": m, "p": p, "L_ns": n}
    n_max = int(L_.mhdg_factor_max_n(1))
    if n > n_max:
        out["status"] = f"not run: L ns > {n_max} (batched LU kernel limit)"
        return out
    case = TgvCase(reynolds=1600.0, mach=0.1)
    gmesh = build_cube_mesh(case.domain, N1D, m, periodic=(True, True, True))
    need = gmesh.n_macro * bytes_per_macro(m, p) + 8 * CHUNK * n * n
    P = 1
    while need / P > BUDGET:
        P *= 2
    out.update(n_macros_total=gmesh.n_macro, est_device_GB_total=need / 1e9, n_gpus_needed=P)
    if P > 8:
        out["status"] = "not run: needs more than 8 GPUs"
        return out
    mesh = gmesh if P == 1 else partition_mesh(gmesh, 0, P).mesh
    disc = Discretization(mesh, p, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    f = A.to_device_fields(disc, u, np.zeros((disc.n_mac, 3, disc.L, 5)), uhat)
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    ctx = A.StageContext.dirk_stage(0.01, S.DirkTableau.dirk33().d[0], 0, [], f.u)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    e0, e1 = ev(), ev()
    if REPR == "recompute":
        blocks = A.RecomputeBlocks(disc, f, ctx, chunk=CHUNK)
        del f
        cond = CondensedRecompute.build(blocks, precond=False)  # assembly + Schur + LU, window by window
        torch.cuda.synchronize()
        e0.record()
        cond.refactor()
        e1.record()
        torch.cuda.synchronize()
    else:
        blocks, _ = A.jacobian(disc, f, ctx)
        del f
        torch.cuda.synchronize()
        cond = CondensedSchur.allocate(blocks, scratch_macros=CHUNK)
        st = disc.device.status_buffer()
        cond.refactor_async(st)
        torch.cuda.synchronize()
        e0.record()
        cond.refactor_async(st)
        e1.record()
        torch.cuda.synchronize()
        A.raise_status(st, "condense")
    t_cond = e0.elapsed_time(e1) / 1e3
    xs = torch.as_tensor(np.random.default_rng(1).standard_normal((4, disc.n_trace)), device="cuda")
    y = torch.empty(disc.n_trace, dtype=torch.float64, device="cuda")
    for i in range(3):
        cond.apply_trace(xs[i], out=y)
    torch.cuda.synchronize()
    with _lib.Timeline(4096) as tl:
        cond.apply_trace(xs[0], out=y)
        torch.cuda.synchronize()
    paths = sorted(k for k in tl.ms if k.startswith("apply") or (REPR == "recompute" and k == "assemble"))
    out["representation"] = REPR
    if REPR == "recompute":
        out["condense_includes"] = "window-wise Jacobian assembly + Schur + LU"
        out["apply_kernels_ms"] = {k: tl.ms[k] for k in paths}
    e0.record()
    for i in range(200):
        cond.apply_trace(xs[i & 3], out=y)
    e1.record()
    torch.cuda.synchronize()
    t_app = e0.elapsed_time(e1) / 1e3 / 200
    b_mac = bench.algorithmic_bytes_per_macro(disc)
    f_mac = bench.condense_flops_per_macro(disc)
    peaks = bench.measured_peaks()
    hbm = float(peaks.get("hbm_gbs", 6533.2))
    out.update(
        status="ok" if P == 1 else f"rank-0 slab of a {P}-GPU partition",
        n_macros_this_gpu=disc.n_mac, n_trace_this_gpu=disc.n_trace, apply_kernels=paths,
        condense_s=t_cond, condense_macros_per_s=disc.n_mac / t_cond,
        condense_tflops_canonical=disc.n_mac * f_mac / t_cond / 1e12,
        apply_s=t_app, apply_dof_per_s=disc.n_trace / t_app,
        apply_GBs_B_ref=disc.n_mac * b_mac / t_app / 1e9, apply_frac_B_ref=disc.n_mac * b_mac / t_app / 1e9 / hbm,
        two_hundred_applies_s=200 * t_app, peak_device_GB=torch.cuda.max_memory_allocated() / 1e9)
    del cond, blocks, disc
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    return out


if __name__ == "__main__":
    combos = [(m, p) for m in (1, 2, 4) for p in (1, 2, 3)]
    if len(sys.argv) > 2:
        combos = [tuple(int(v) for v in c.split(",")) for c in sys.argv[2:]]
    for m, p in combos:
        t0 = time.perf_counter()
        try:
            r = run(m, p)
        except Exception as exc:  # report and continue the sweep
            r = {"m": m, "p": p, "status": f"error: {type(exc).__name__}: {exc}"[:300]}
            torch.cuda.empty_cache()
        r["wall_s"] = time.perf_counter() - t0
        print(json.dumps(r), flush=True)
