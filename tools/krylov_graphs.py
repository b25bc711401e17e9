"""C1 (BASELINE configs[0]) Krylov latency with and without the CUDA-graph-captured
Arnoldi steps (krylov._StepGraphs): one solve_trace_system at the seeded C1 state,
then the whole PTC + FGMRES run to 1e-10.  Prints one JSON line per setting."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import load_golden  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import krylov as K  # noqa: E402
from paper_2402_11361_b200 import stepper as S  # noqa: E402
from paper_2402_11361_b200.cases import CouettePlane2D  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_square_mesh  # noqa: E402

g = load_golden("c1_ptc_oracle")
case = CouettePlane2D()
d = Discretization(build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False)), 2, case.params,
                   bcs=case.boundary_conditions())
for on in [False, True] * 2:  # the first pair warms up the library and the allocator
    K.KRYLOV_GRAPHS = on
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    blocks, _ = A.jacobian(d, f, A.StageContext.steady(1.0))
    cond = CondensedSchur.build(blocks)
    b = torch.as_tensor(np.random.default_rng(3).standard_normal(d.n_trace), device="cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res, nmv = K.solve_trace_system(cond, b, K.KrylovConfig(rel_tol=1e-10, max_iter=400), "fgmres")
    torch.cuda.synchronize()
    t_solve = time.perf_counter() - t0
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st, _ = S.ptc_steady_solve(d, f, rel_tol=1e-10)
    torch.cuda.synchronize()
    t_ptc = time.perf_counter() - t0
    print(json.dumps({"graphs": on, "solve_s": round(t_solve, 4), "solve_fgmres_iters": res.iterations,
                      "solve_matvecs": nmv, "us_per_matvec": round(1e6 * t_solve / nmv, 1),
                      "ptc_s": round(t_ptc, 3), "newton": st.iterations, "krylov": st.krylov_iterations,
                      "final_residual": st.residuals[-1]}), flush=True)
