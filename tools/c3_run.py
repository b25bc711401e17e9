"""BASELINE configs[2] (C3) end to end on one B200: 3D Taylor-Green vortex, Re=1600,
M=0.1, periodic [-pi, pi]^3, 16^3 hexes x 6 = 24,576 macros, m=2, p=2, 10 steps of
DIRK(3,3) with dt = 0.01, Newton + block-preconditioned FGMRES per stage, through the
reference's driver API (stepper.dirk_advance, stepper.py:265-328; TgvCase,
cases.py:110-158).  Writes per-stage Newton/FGMRES/matvec counts, phase times and a
kinetic-energy trace to profiles/r2_c3_run.json.

    python tools/c3_run.py [steps] [n_ele_1d]
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import stepper as S  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402


def kinetic_energy(disc, u):
    """Volume-weighted mean of rho |v|^2 / 2 (nodal mass-matrix quadrature)."""
    M = torch.as_tensor(disc.rm.mass, device=u.device)
    det = torch.as_tensor(disc.det, device=u.device)
    rho = u[..., 0]
    ke = 0.5 * (u[..., 1:4] ** 2).sum(-1) / rho
    tot = torch.einsum("mi,ij,m->", ke, M, det) / torch.einsum("ij,m->", M, det)
    return float(tot)


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n1d = int(sys.argv[2]) if len(sys.argv) > 2 else 16
    torch.cuda.set_device(0)
    case = TgvCase(reynolds=1600.0, mach=0.1)
    t0 = time.perf_counter()
    disc = Discretization(build_cube_mesh(case.domain, n1d, 2, periodic=(True, True, True)), 2, case.params)
    u, uhat = disc.nodal_interpolant(case.initial_state)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(disc, f.u, f.uhat)
    t_setup = time.perf_counter() - t0
    tab = S.DirkTableau.dirk33()
    out = dict(config="C3: TGV Re=1600 M=0.1, %d^3 x 6 = %d macros, m=2, p=2, DIRK33 dt=0.01" % (n1d, disc.n_mac),
               n_mac=disc.n_mac, n_trace=disc.n_trace, setup_s=t_setup, steps=[],
               device=torch.cuda.get_device_name(0), ke0=kinetic_energy(disc, f.u))
    print(out["config"], flush=True)
    for k in range(steps):
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        with _lib.Timeline(1 << 16) as tl:
            sts, dt = S.dirk_advance(disc, f, 0.01, tab)
            torch.cuda.synchronize()
        wall = time.perf_counter() - s0
        rec = dict(step=k + 1, dt=dt, wall_s=wall, ke=kinetic_energy(disc, f.u),
                   newton=[s.iterations for s in sts], fgmres=[s.krylov_iterations for s in sts],
                   matvecs=[s.krylov_matvecs for s in sts], residuals=[s.residuals for s in sts],
                   timings={key: sum(s.timings[key] for s in sts) for key in sts[0].timings},
                   kernel_ms={key: tl.ms[key] for key in tl.ms}, kernel_counts=dict(tl.counts))
        out["steps"].append(rec)
        print(json.dumps({k2: rec[k2] for k2 in ("step", "wall_s", "ke", "newton", "fgmres", "matvecs")}),
              flush=True)
    out["total_wall_s"] = sum(r["wall_s"] for r in out["steps"])
    out["totals"] = {key: sum(r["timings"][key] for r in out["steps"]) for key in out["steps"][0]["timings"]}
    out["kernel_ms_total"] = {}
    for r in out["steps"]:
        for key, v in r["kernel_ms"].items():
            out["kernel_ms_total"][key] = out["kernel_ms_total"].get(key, 0.0) + v
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    repr_ = os.environ.get("MHDG_APPLY_REPR", "matrix_free")
    out["representation"] = repr_
    out["peak_device_GB"] = torch.cuda.max_memory_allocated() / 1e9
    path = os.path.join(ROOT, "gpurun_out", "r2_c3_run.json" if repr_ == "matrix_free" else f"r2_c3_run_{repr_}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print("total", out["total_wall_s"], out["totals"], flush=True)


if __name__ == "__main__":
    main()
