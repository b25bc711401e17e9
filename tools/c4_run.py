"""C4 (flow past a sphere, BASELINE configs[3]) on one B200: the O-grid's inner
N_R radial shells (grading 1.15 from r = 0.5, the full 24 polar x 48 azimuthal
cells, pole wedges), m = 2, p = 2, Re = 100, M = 0.2, adiabatic no-slip sphere,
free-stream far field at the truncated outer radius; free stream + U(-1e-3,
1e-3) (seed 0); 5 PTC Newton steps with FGMRES.  The full 32 shells (211,968
macros, ~1.8 MB of device data per macro) need two or more GPUs (slabs of
shells, bench.py / dist.py); one GPU holds the inner ~12.

    python tools/c4_run.py [N_R] [max_newton]   (defaults 12, 5)

With MHDG_APPLY_REPR=recompute (the coupling-recompute representation, B_min: only the S
factors and the face preconditioner resident) the full 32 shells fit one B200:
    MHDG_APPLY_REPR=recompute python tools/c4_run.py 32
Each Newton step appends one JSON line to gpurun_out/c4_steps.jsonl as it completes.
"""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import stepper as S  # noqa: E402
from paper_2402_11361_b200.cases import SphereCase  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_sphere_ogrid_mesh  # noqa: E402

n_r = int(sys.argv[1]) if len(sys.argv) > 1 else 12
max_newton = int(sys.argv[2]) if len(sys.argv) > 2 else 5
REPR = os.environ.get("MHDG_APPLY_REPR", "matrix_free")
STEPS = os.path.join(ROOT, "gpurun_out", "c4_steps.jsonl")
w = 1.15 ** np.arange(32)
r_full = 0.5 + 19.5 * np.concatenate([[0.0], np.cumsum(w)]) / np.sum(w)
case = SphereCase()
T0 = time.perf_counter()


def log(msg):
    print(f"[{time.perf_counter() - T0:8.1f} s] {msg}", flush=True)


t0 = time.perf_counter()
mesh = build_sphere_ogrid_mesh(n_r, 24, 48, 2, r_in=0.5, r_out=float(r_full[n_r]))
log(f"mesh: {mesh.n_macro} macros")
disc = Discretization(mesh, 2, case.params, bcs=case.boundary_conditions())
log("discretization")
u, uhat = disc.nodal_interpolant(case.freestream)
rng = np.random.default_rng(0)
u = u + rng.uniform(-1e-3, 1e-3, u.shape)
uhat = uhat + rng.uniform(-1e-3, 1e-3, uhat.shape)
f = A.to_device_fields(disc, u, np.zeros((disc.n_mac, 3, disc.L, 5)), uhat)
f.q = A.gradient_refresh(disc, f.u, f.uhat)
torch.cuda.synchronize()
t_setup = time.perf_counter() - t0
log("device state")
ptc = S.PtcState(dtau=1.0, tau_init=1.0, tau_max=1e8)
t0 = time.perf_counter()


def on_step(s):
    log(f"newton {s.iterations}: residual {s.residuals[-1]:.4e}, krylov {s.krylov_iterations}")
    os.makedirs(os.path.dirname(STEPS), exist_ok=True)
    with open(STEPS, "a") as fh:
        fh.write(json.dumps({"n_macros": disc.n_mac, "representation": REPR, "newton": s.iterations,
                             "residuals": [float(r) for r in s.residuals], "dtau": [float(x) for x in s.dtau],
                             "krylov_iterations": s.krylov_iterations, "krylov_matvecs": s.krylov_matvecs,
                             "seconds_since_start": time.perf_counter() - t0,
                             "timings": {k: float(v) for k, v in s.timings.items()},
                             "peak_device_GB": torch.cuda.max_memory_allocated() / 1e9}) + "\n")


st = S.newton_solve(disc, f, A.StageContext.steady(), max_newton=max_newton, ptc=ptc, abs_tol=1e-10, rel_tol=1e-10,
                    log=on_step)
torch.cuda.synchronize()
t_run = time.perf_counter() - t0
print(json.dumps({
    "config": f"C4 inner {n_r} of 32 shells (r_out {r_full[n_r]:.3f}), 24 x 48 cells, m=2, p=2",
    "representation": REPR,
    "n_macros": disc.n_mac, "n_trace_dofs": disc.n_trace, "newton": st.iterations,
    "krylov_iterations": st.krylov_iterations, "krylov_matvecs": st.krylov_matvecs,
    "residuals": [float(r) for r in st.residuals], "dtau": [float(x) for x in st.dtau],
    "seconds": {"setup_host": t_setup, "newton_total": t_run, **{k: float(v) for k, v in st.timings.items()}},
    "peak_device_GB": torch.cuda.max_memory_allocated() / 1e9}))
