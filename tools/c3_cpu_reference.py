"""CPU baseline for C3: the REFERENCE (/root/reference, pure numpy/numba) timed on a
384-macro slab subset (TGV, n_ele_1d=4 -> 4^3 x 6 macros, m=2, p=2, DIRK33 stage-1
context) -- residual, Jacobian, condensation (schur) and 10 applies, as SURVEY 8d
prescribes; per-macro and per-DOF rates are intensive.  Runs in the build container
only (the GPU box has no /root/reference).  Thread count is pinned to 1 (the
reference's c_einsum is single threaded; SURVEY 6.2 measured 8 threads no faster).

    OPENBLAS_NUM_THREADS=1 NUMBA_NUM_THREADS=1 python tools/c3_cpu_reference.py
"""
import json
import os
import platform
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
import numpy as np  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/src")
import macrohdg.assembly as RA  # noqa: E402
import macrohdg.condense as RC  # noqa: E402
import macrohdg.stepper as RS  # noqa: E402
from macrohdg.cases import TgvCase  # noqa: E402
from macrohdg.mesh import build_cube_mesh  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    tgv = TgvCase(reynolds=1600, mach=0.1)
    rd = RA.Discretization(build_cube_mesh(tgv.domain, n1d, 2, periodic=(True,) * 3), 2, tgv.params)
    f = rd.interpolate(tgv.initial_state)
    tab = RS.DirkTableau.dirk33()
    ctx = RA.StageContext.dirk_stage(0.01, tab.d[0], 0, [], f.u)
    RA.residual(rd, f, ctx)  # JIT warm-up
    t = {}
    t0 = time.perf_counter()
    res = RA.residual(rd, f, ctx)
    t["residual"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    blocks, _ = RA.jacobian(rd, f, ctx)
    t["jacobian"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    cond = RC.condense(blocks, "schur")
    t["condense"] = time.perf_counter() - t0
    x = np.random.default_rng(1).standard_normal(rd.n_trace)
    n_apply = 10
    t0 = time.perf_counter()
    for _ in range(n_apply):
        cond.apply_trace(x)
    t["apply"] = (time.perf_counter() - t0) / n_apply
    M = rd.n_mac
    out = dict(what="reference (macrohdg, /root/reference) CPU rates, C3 shape (m=2, p=2), TGV DIRK33 stage-1 context",
               sample=f"{n1d}^3 x 6 = {M} macros, {rd.n_trace} trace dofs", threads=1, cpu=platform.processor() or
               platform.machine(), host="build container (the GPU box has no /root/reference)",
               seconds=t, residual_mac_per_s=M / t["residual"], jacobian_mac_per_s=M / t["jacobian"],
               condense_mac_per_s=M / t["condense"], apply_dof_per_s=rd.n_trace / t["apply"],
               c3_extrapolation_s={"jacobian": 24576 / (M / t["jacobian"]), "condense": 24576 / (M / t["condense"]),
                                   "apply": 3686400 / (rd.n_trace / t["apply"])})
    path = os.path.join(ROOT, "profiles", "r2_c3_reference_cpu_rates.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
