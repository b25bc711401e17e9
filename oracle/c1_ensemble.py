"""Sensitivity of the C1 PTC run (BASELINE configs[0]) to rounding-level noise.

Test infrastructure (evidence for the tolerances of tests/test_gpu_drivers.py).
Every Newton step after the first ends at FGMRES's 400-iteration cap with the
linear system unconverged, so the Krylov solution -- and with it the PTC
trajectory -- amplifies rounding differences: the oracle's own explicit-inverse
and LU-solve runs (two backward-stable factorizations, solves accurate to 1e-14)
differ by 7e-7 in the state after step 2.  This script reruns the oracle (LU
mode) from the C1 initial state perturbed by uniform noise of relative size
1e-14 (seeds 1..K) and records Newton/FGMRES counts, per-step residuals and the
final-state spread against tests/golden/c1_ptc_oracle_lu.npz.

    python oracle/c1_ensemble.py SEED  -> profiles/r2_c1_ensemble_SEED.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle.hdg_oracle as O  # noqa: E402
from oracle.make_c1_golden import c1_setup  # noqa: E402


def main(seed):
    case, disc, u, uhat = c1_setup()
    rng = np.random.default_rng(1000 + seed)
    u = u * (1.0 + 1e-14 * rng.uniform(-1, 1, u.shape))
    uhat = uhat * (1.0 + 1e-14 * rng.uniform(-1, 1, uhat.shape))
    q = O.gradient_refresh(disc, u, uhat)
    f = O.Fields(u, q, uhat)
    t0 = time.perf_counter()
    st, _ = O.ptc_steady_solve(disc, f, rel_tol=1e-10, mode="lu")
    g = np.load(os.path.join(ROOT, "tests", "golden", "c1_ptc_oracle_lu.npz"))
    rho_ratio = f.u[..., 0] / g["u"][..., 0]
    out = dict(seed=seed, ic_noise=1e-14, newton=st.iterations, krylov=st.krylov_iterations,
               krylov_per_step=st.krylov_per_step, residuals=st.residuals,
               final_u_rel_diff=float(np.abs(f.u - g["u"]).max() / np.abs(g["u"]).max()),
               final_rho_offset=float(rho_ratio.mean() - 1.0), final_rho_ratio_spread=float(rho_ratio.std()),
               seconds=time.perf_counter() - t0)
    path = os.path.join(ROOT, "profiles", f"r2_c1_ensemble_{seed}.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]))
