"""One Newton step's Krylov phase at C3 (24,576 macros, DIRK33 stage-1 context): the
condensed rhs and the FGMRES(inner GMRES) solve with the block preconditioner, inside an
NVTX range "krylov" -- for the ncu launch list showing which kernels run there
(no cuBLAS / torch reductions on the trace vectors).

    ncu --nvtx --nvtx-include "krylov/" --metrics gpu__time_duration.sum --csv \
        --log-file OUT python tools/prof_krylov.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import krylov as K  # noqa: E402
from paper_2402_11361_b200.cases import TgvCase  # noqa: E402
from paper_2402_11361_b200.condense import condense  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_cube_mesh  # noqa: E402
from paper_2402_11361_b200.stepper import DirkTableau  # noqa: E402

n1d = int(sys.argv[1]) if len(sys.argv) > 1 else 16
case = TgvCase(reynolds=1600.0, mach=0.1)
disc = Discretization(build_cube_mesh(case.domain, n1d, 2, periodic=(True,) * 3), 2, case.params)
u, uhat = disc.nodal_interpolant(case.initial_state)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
ctx = A.StageContext.dirk_stage(0.01, DirkTableau.dirk33().d[0], 0, [], f.u)
res = A.residual(disc, f, ctx)
blocks, _ = A.jacobian(disc, f, ctx)
cond = condense(blocks)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("krylov")
b = cond.rhs(*res)
r, nmv = K.solve_trace_system(cond, b, K.KrylovConfig(rel_tol=1e-8), "fgmres")
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print(f"C3 Krylov phase: {r.iterations} FGMRES iterations, {nmv} matvecs, converged {r.converged}")
