"""Multi-rank path on CPU: 2 processes over gloo run the real slab partition,
halo plans, communicator, distributed condensed operator (forward + reverse
halo), distributed residual trace sum, and distributed FGMRES/GMRES with the
face-block preconditioner whose shared faces get the neighbour's block --
with oracle-backed local operators -- and must reproduce the single-process
oracle (only summation order may change)."""

import os
import socket

import numpy as np
import pytest
import scipy.linalg
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleLocal:
    """Local operator of one slab backed by the oracle (numpy) on CPU tensors."""

    def __init__(self, cond):
        self.cond = cond
        self.blocks = cond.blocks

    def apply_trace(self, x):
        return torch.from_numpy(self.cond.apply_trace(x.numpy()))

    def rhs(self, R_Q, R_U, R_T):
        return torch.from_numpy(self.cond.rhs(R_Q.numpy(), R_U.numpy(), R_T.numpy()))

    def recover(self, R_Q, R_U, x):
        du, dq = self.cond.recover(R_Q.numpy(), R_U.numpy(), x.numpy())
        return torch.from_numpy(du), torch.from_numpy(dq)


def _side_blocks(disc, blocks, faces_local):
    """Canonical P^T FTT P of the local side of each given local face (numpy)."""
    bs = disc.Lf * disc.ns
    fo, so = disc.mesh.faces_of_macro, disc.mesh.sides_of_macro
    where = {}
    for mac in range(disc.n_mac):
        for lf in range(disc.nf):
            where.setdefault(int(fo[mac, lf]), (mac, lf))
    out = np.zeros((len(faces_local), bs, bs))
    for i, f in enumerate(faces_local):
        mac, lf = where[int(f)]
        pi = disc.gather[mac, lf] - f * bs
        out[i][np.ix_(pi, pi)] = blocks.face_trace_trace[mac, lf]
    return out


def _dist_precond(dd, comm, blocks):
    import oracle.hdg_oracle as O

    disc, part = dd.local, dd.part
    bs = disc.Lf * disc.ns
    sends = {q: torch.from_numpy(_side_blocks(disc, blocks, f).ravel()) for q, f in part.recv_faces.items()}
    got = comm.exchange(sends, {q: len(f) * bs * bs for q, f in part.send_faces.items()}, torch.zeros(1, dtype=torch.float64))
    B = np.zeros((part.n_local_faces, bs, bs))
    fo = disc.mesh.faces_of_macro
    pi = disc.gather.reshape(disc.n_mac, disc.nf, bs) - fo[:, :, None] * bs
    np.add.at(B, (fo[:, :, None, None], pi[:, :, :, None], pi[:, :, None, :]), blocks.face_trace_trace)
    for q, buf in got.items():
        B[part.send_faces[q]] += buf.numpy().reshape(-1, bs, bs)
    B = 0.5 * (B + np.swapaxes(B, -1, -2))
    nown = part.n_owned_faces
    inv = np.stack([scipy.linalg.cho_solve((np.linalg.cholesky(B[f]), True), np.eye(bs)) for f in range(nown)])
    del O
    return lambda v: torch.from_numpy(np.matmul(inv, v.numpy().reshape(nown, bs, 1)).reshape(-1))


def _worker(rank, world, port, q):
    import sys

    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle.hdg_oracle as O
        from paper_2402_11361_b200 import krylov as K
        from paper_2402_11361_b200.cases import CouettePlane2D
        from paper_2402_11361_b200.discretization import Discretization
        from paper_2402_11361_b200.dist import Comm, DistCondensed, DistDiscretization
        from paper_2402_11361_b200.mesh import build_square_mesh

        case = CouettePlane2D()
        gmesh = build_square_mesh(case.domain, (4, 2), 2, periodic=(True, False))
        gd = Discretization(gmesh, 1, case.params, bcs=case.boundary_conditions())
        f = O.interpolate(gd, case.exact_state)
        rng = np.random.default_rng(0)
        f.u = f.u * (1 + 1e-3 * rng.standard_normal(f.u.shape))
        f.uhat = f.uhat * (1 + 1e-3 * rng.standard_normal(f.uhat.shape))
        ctx = O.Ctx.steady(4.0)
        gres = O.residual(gd, f, ctx)
        gblocks, _ = O.jacobian(gd, f, ctx)
        gcond = O.condense(gblocks)

        comm = Comm()
        # a one-sided exchange (a rank that owns every shared face only sends): rank 0 -> rank 1
        peer = 1 - rank
        sends = {peer: torch.arange(3, dtype=torch.float64)} if rank == 0 else {}
        recv = {peer: torch.empty(3, dtype=torch.float64)} if rank == 1 else {}
        comm.exchange_start(sends, recv)()
        if rank == 1:
            assert recv[peer].tolist() == [0.0, 1.0, 2.0]
        dd = DistDiscretization(gmesh, 1, case.params, bcs=case.boundary_conditions(), comm=comm,
                                plan_device=torch.device("cpu"))
        part, disc = dd.part, dd.local
        lo, hi = part.macro_range
        own = part.global_dofs_owned(disc.Lf, disc.ns)
        loc = part.global_dofs_local(disc.Lf, disc.ns)
        lf_ = O.Fields(f.u[lo:hi], f.q[lo:hi], f.uhat[loc])
        # residual: local trace sums + reverse halo == global residual on owned dofs
        R_Q, R_U, R_Tl = O.residual(disc, lf_, ctx)
        R_T = dd.reverse(torch.from_numpy(R_Tl)).numpy()
        res = {"R_U": float(np.max(np.abs(R_U - gres[1][lo:hi]))),
               "R_T": float(np.max(np.abs(R_T - gres[2][own])) / np.max(np.abs(gres[2])))}
        lblocks, _ = O.jacobian(disc, lf_, ctx)
        res["blocks"] = float(np.max(np.abs(lblocks.state_state - gblocks.state_state[lo:hi])))
        dcond = DistCondensed(dd, OracleLocal(O.condense(lblocks)))
        x = np.random.default_rng(5).standard_normal(gd.n_trace)
        y = dcond.apply_trace(torch.from_numpy(x[own])).numpy()
        yg = gcond.apply_trace(x)
        res["apply"] = float(np.max(np.abs(y - yg[own])) / np.max(np.abs(yg)))
        b = dcond.rhs(torch.from_numpy(R_Q), torch.from_numpy(R_U), torch.from_numpy(R_T)).numpy()
        bg = gcond.rhs(*gres)
        res["rhs"] = float(np.max(np.abs(b - bg[own])) / np.max(np.abs(bg)))
        du, _ = dcond.recover(torch.from_numpy(R_Q), torch.from_numpy(R_U), torch.from_numpy(x[own]))
        dug, _ = gcond.recover(gres[0], gres[1], x)
        res["recover"] = float(np.max(np.abs(du.numpy() - dug[lo:hi])) / np.max(np.abs(dug)))
        # distributed Krylov with the split-face preconditioner
        pre = _dist_precond(dd, comm, lblocks)
        gpre = O.block_precond_build(gcond)
        res["precond"] = float(np.max(np.abs(pre(torch.from_numpy(x[own])).numpy() - gpre(x)[own])))
        cfg = K.KrylovConfig(rel_tol=1e-8)
        icfg = K.KrylovConfig(restart=20, max_iter=20, rel_tol=0.1)
        r = K.fgmres(dcond.apply_trace, torch.from_numpy(bg[own]),
                     lambda v: K.gmres(dcond.apply_trace, v, precond=pre, cfg=icfg, comm=comm).x, cfg=cfg, comm=comm)
        og = O.solve_trace_system(gcond, bg, O.KrylovConfig(rel_tol=1e-8), "fgmres")[0]
        res["fgmres_iters"] = (r.iterations, og.iterations)
        res["fgmres_x"] = float(np.max(np.abs(r.x.numpy() - og.x[own])) / np.max(np.abs(og.x)))
        res["n_owned"] = part.n_owned_faces
        res["n_global_faces"] = gmesh.n_faces
        res["n_ghost"] = part.n_ghost_faces
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


def test_two_rank_slab_operator_and_krylov():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    print(out)
    assert sum(r["n_ghost"] for r in out.values()) > 0, out
    for rank, r in out.items():
        assert r["blocks"] < 1e-13, (rank, r)
        assert r["R_U"] < 1e-12 and r["R_T"] < 1e-12, (rank, r)
        assert r["apply"] < 1e-12, (rank, r)
        assert r["rhs"] < 1e-10 and r["recover"] < 1e-10, (rank, r)
        assert r["precond"] < 1e-12, (rank, r)
        assert sum(x["n_owned"] for x in out.values()) == r["n_global_faces"]
        it, git = r["fgmres_iters"]
        assert abs(it - git) <= 1, (rank, r)
        assert r["fgmres_x"] < 1e-7, (rank, r)
