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
from paper_2402_11361_b200 import condense as CD  # noqa: E402

for on, repr_ in [(False, "matrix_free"), (True, "matrix_free")] * 2 + [(True, "auto"), (False, "auto")]:
    K.KRYLOV_GRAPHS = on
    CD.APPLY_REPR = repr_
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
    print(json.dumps({"graphs": on, "apply_repr": repr_, "solve_s": round(t_solve, 4), "solve_fgmres_iters": res.iterations,
                      "solve_matvecs": nmv, "us_per_matvec": round(1e6 * t_solve / nmv, 1),
                      "ptc_s": round(t_ptc, 3), "newton": st.iterations, "krylov": st.krylov_iterations,
                      "final_residual": st.residuals[-1]}), flush=True)

# breakdown of one inner step at C1: graph replay + sync, host Givens, eager pieces
K.KRYLOV_GRAPHS = True
CD.APPLY_REPR = "matrix_free"
cond.ahat = None
op, cnt = K.make_counted(cond.apply_trace, capturable=True)
pre = K.block_precond_build(cond)
ws = K._StepGraphs(20, d.n_trace, b.device, cnt, False)
V = ws.V
V.copy_(torch.randn_like(V))
body = lambda i: K._icgs_launch(V, i, pre(op(V[i])))  # noqa: E731
for j in range(8):
    ws.run(j, body)
torch.cuda.synchronize()


def tm(fn, reps=500):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return round(1e6 * (time.perf_counter() - t0) / reps, 1)


g7 = ws.graphs[7][0]
out = ws.graphs[7][1][1]
H = np.random.rand(21, 20)
cs, sn, gg = np.zeros(20), np.zeros(20), np.zeros(21)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    g7.replay()
e1.record()
torch.cuda.synchronize()
print(json.dumps({
    "replay_only_us": tm(lambda: g7.replay()),
    "replay_gpu_us_back_to_back": round(1e3 * e0.elapsed_time(e1) / 200, 1),
    "replay_fetch_us": tm(lambda: (g7.replay(), K._icgs_fetch(out, 7, d.n_trace))),
    "eager_step_fetch_us": tm(lambda: K._icgs_fetch(body(7)[1], 7, d.n_trace)),
    "apply_eager_us": tm(lambda: op(V[3])),
    "precond_eager_us": tm(lambda: pre(V[3])),
    "givens_j10_us": tm(lambda: K._givens(H, cs, sn, gg, 10)),
    "v_update_us": tm(lambda: V.__setitem__(9, V[8] / 1.7)),
}), flush=True)
