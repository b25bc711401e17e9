"""Per-iteration cost of the Krylov building blocks at C1 and C2 sizes: apply,
block preconditioner, ICGS (torch), and the host sync of the Hessenberg column."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import bench  # noqa: E402
from paper_2402_11361_b200 import assembly as A  # noqa: E402
from paper_2402_11361_b200 import krylov as K  # noqa: E402
from paper_2402_11361_b200.cases import CouettePlane2D  # noqa: E402
from paper_2402_11361_b200.condense import CondensedSchur  # noqa: E402
from paper_2402_11361_b200.discretization import Discretization  # noqa: E402
from paper_2402_11361_b200.mesh import build_square_mesh  # noqa: E402


def setup(name):
    if name == "C1":
        case = CouettePlane2D()
        d = Discretization(build_square_mesh(case.domain, (8, 4), 2, periodic=(True, False)), 2, case.params,
                           bcs=case.boundary_conditions())
        u, uhat = d.nodal_interpolant(case.exact_state)
    else:
        case, d = bench.c2_discretization()
        u, uhat = bench.c2_state(case, d)
    f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    f.q = A.gradient_refresh(d, f.u, f.uhat)
    blocks, _ = A.jacobian(d, f, A.StageContext.steady(1.0))
    return d, CondensedSchur.build(blocks)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


for name, reps in (("C1", 2000), ("C2", 50)):
    d, cond = setup(name)
    pre = K.block_precond_build(cond)
    x = torch.randn(d.n_trace, dtype=torch.float64, device="cuda")
    V = torch.randn(31, d.n_trace, dtype=torch.float64, device="cuda")
    w = torch.randn(d.n_trace, dtype=torch.float64, device="cuda")
    print(f"{name}: n_trace {d.n_trace}")
    print(f"  apply_trace      {timeit(lambda: cond.apply_trace(x), reps):9.1f} us")
    print(f"  precond          {timeit(lambda: pre(x), reps):9.1f} us")
    print(f"  icgs j=15 (host) {timeit(lambda: K._icgs_host(V, 15, w), reps):9.1f} us")
    print(f"  sync + .cpu()    {timeit(lambda: w[:2].cpu(), reps):9.1f} us")
    b = cond.apply_trace(x)
    cfg = K.KrylovConfig(restart=20, max_iter=20, rel_tol=1e-30, abs_tol=1e-300)
    t = timeit(lambda: K.gmres(cond.apply_trace, b, precond=pre, cfg=cfg), max(2, reps // 40))
    print(f"  gmres(20) total  {t:9.1f} us = {t / 20:.1f} us per iteration")
