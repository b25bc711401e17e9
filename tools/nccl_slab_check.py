"""One rank of the NCCL slab check (tests/test_gpu_nccl.py), launched by torchrun:
the distributed apply and an FGMRES solve on 2D uniform flow, each rank its own
GPU, compared with the single-process run on the same GPU.

    python -m torch.distributed.run --standalone --nproc-per-node 2 tools/nccl_slab_check.py OUTDIR
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _worker(rank, world, out_dir):
    import torch.distributed as dist

    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200 import krylov as K
    from paper_2402_11361_b200.cases import UniformFlow2D
    from paper_2402_11361_b200.condense import condense
    from paper_2402_11361_b200.discretization import Discretization
    from paper_2402_11361_b200.dist import DistDiscretization
    from paper_2402_11361_b200.mesh import build_square_mesh

    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world)
    case = UniformFlow2D()
    mesh = build_square_mesh(case.domain, (8 * world, 4), 2, periodic=(True, True))
    gd = Discretization(mesh, 2, case.params)
    u, uhat = gd.nodal_interpolant(case.state)
    rng = np.random.default_rng(0)
    u = u * (1 + 1e-3 * rng.standard_normal(u.shape))
    gf = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
    gf.q = A.gradient_refresh(gd, gf.u, gf.uhat)
    ctx = A.StageContext.steady(1.0)
    x = torch.as_tensor(rng.standard_normal(gd.n_trace), device="cuda")
    gcond = condense(A.jacobian(gd, gf, ctx)[0])
    y_ref = gcond.apply_trace(x)
    r_ref, _ = K.solve_trace_system(gcond, x, K.KrylovConfig(rel_tol=1e-8), "fgmres")

    dd = DistDiscretization(mesh, 2, case.params)
    lo, hi = dd.part.macro_range
    own = torch.as_tensor(dd.owned_global_dofs(), device="cuda")
    f = A.FieldState(gf.u[lo:hi].clone(), gf.q[lo:hi].clone(), gf.uhat[own].clone())
    cond = condense(A.jacobian(dd, f, ctx)[0])
    y = cond.apply_trace(x[own].clone())
    r, _ = K.solve_trace_system(cond, x[own].clone(), K.KrylovConfig(rel_tol=1e-8), "fgmres")
    torch.cuda.synchronize()
    res = dict(apply_equal=bool(torch.equal(y, y_ref[own])),
               iters=(r.iterations, r_ref.iterations),
               x_err=float((r.x - r_ref.x[own]).abs().max() / r_ref.x.abs().max()))
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), res, allow_pickle=True)
    dist.destroy_process_group()



if __name__ == "__main__":
    _worker(int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), sys.argv[1])
