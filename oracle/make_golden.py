"""Generate tests/golden/*.npz by running the REFERENCE implementation.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python -m oracle.make_golden

Every fixture stores the inputs (seeded) together with the reference's
outputs, so tests can pin both the oracle restatement and the CUDA path to
the reference without the reference being present.  Versions of the
third-party numerics used are recorded in each file.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def _versions():
    import numba
    import scipy

    return np.array(f"numpy {np.__version__}; scipy {scipy.__version__}; numba {numba.__version__}")


def _perturbed(rd, fields, seed):
    rng = np.random.default_rng(seed)
    fields.u += 1e-3 * rng.standard_normal(fields.u.shape) * np.abs(fields.u).max()
    fields.uhat += 1e-3 * rng.standard_normal(fields.uhat.shape) * np.abs(fields.uhat).max()
    fields.q += 1e-2 * rng.standard_normal(fields.q.shape)
    return rng


def operator_case(name, case, domain, n, m, p, periodic, bcs, source, ctx_kind, full_blocks, seed=0):
    import macrohdg.assembly as RA
    import macrohdg.condense as RC
    import macrohdg.krylov as RK
    from macrohdg.mesh import build_cube_mesh

    rd = RA.Discretization(build_cube_mesh(domain, n, m, periodic=periodic), p, case.params, bcs=bcs,
                           source=source)
    fn = case.initial_state if hasattr(case, "initial_state") else case.exact_state
    f = rd.interpolate(fn)
    rng = _perturbed(rd, f, seed)
    if ctx_kind == "dirk":
        hist = -1.1 * 0.3 * f.u
        ctx = RA.StageContext(50.0, hist, np.inf, 0.02)
    else:
        hist = np.zeros(0)
        ctx = RA.StageContext(0.0, None, 1.0, 1.0)
    res = RA.residual(rd, f, ctx)
    blocks, frozen = RA.jacobian(rd, f, ctx)
    cond = RC.condense(blocks, "schur")
    xs = rng.standard_normal((2, rd.n_trace))
    ys = np.stack([cond.apply_trace(x) for x in xs])
    b = cond.rhs(*res)
    du, dq = cond.recover(res[0], res[1], xs[0])
    pre = RK.block_precond_build(cond)
    out = dict(
        versions=_versions(), n_ele=n, m=m, p=p, periodic=np.array(periodic), ctx_kind=np.array(ctx_kind),
        dt_coeff=ctx.dt_coeff, pseudo_dt=ctx.pseudo_dt, supg_dt=ctx.supg_dt, hist=hist,
        u=f.u, q=f.q, uhat=f.uhat, R_Q=res[0], R_U=res[1], R_T=res[2],
        x=xs, y=ys, rhs=b, rec_du=du, rec_dq=dq, precond_y=pre(xs[0]),
        gather=rd.gather, face_macros=rd.mesh.face_macros, corner_map=rd.mesh.corner_map,
        normals=rd.normals, areas=rd.areas, det=rd.det, h_sub=rd.h_sub,
    )
    S = blocks.state_state - RC._schur_correction(blocks)
    # seeded probe for S and S^-1 (kept separate from the trace x vectors)
    probe = np.random.default_rng(seed + 100).standard_normal((S.shape[0], S.shape[1]))
    out["schur_probe"] = probe
    out["schur_times_probe"] = np.einsum("mab,mb->ma", S, probe)
    out["schur_inv_times_probe"] = np.einsum("mab,mb->ma", cond.schur_inv, probe)
    keys = ["state_state", "face_state_trace", "face_trace_state", "face_trace_trace", "wdgdq_vol",
            "wdgdq_face", "trace_face_scale"]
    for k in keys:
        arr = getattr(blocks, k)
        out[f"blk_{k}"] = arr if full_blocks else arr[:1]
        out[f"sum_{k}"] = arr.reshape(arr.shape[0], -1).sum(axis=1)
        out[f"sq_{k}"] = (arr.reshape(arr.shape[0], -1) ** 2).sum(axis=1)
    out["frz_supg_tau"] = frozen.supg_tau
    out["frz_face_visc_state"] = frozen.face_visc_state
    if full_blocks:
        out["dense_A"] = RC.dense_trace_operator(blocks)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, {k: v.shape for k, v in out.items() if hasattr(v, "shape") and v.size > 1000})


def krylov_case(name, case, n, m, p, seed=0):
    import macrohdg.assembly as RA
    import macrohdg.condense as RC
    import macrohdg.krylov as RK
    from macrohdg.mesh import build_cube_mesh

    rd = RA.Discretization(build_cube_mesh(case.domain, n, m, periodic=(True,) * 3), p, case.params)
    f = rd.interpolate(case.initial_state)
    rng = _perturbed(rd, f, seed)
    hist = -1.1 * 0.3 * f.u
    ctx = RA.StageContext(50.0, hist, np.inf, 0.02)
    res = RA.residual(rd, f, ctx)
    blocks, _ = RA.jacobian(rd, f, ctx)
    cond = RC.condense(blocks, "schur")
    b = cond.rhs(*res)
    out = dict(versions=_versions(), n_ele=n, m=m, p=p, u=f.u, q=f.q, uhat=f.uhat, hist=hist, rhs=b)
    for solver in ("fgmres", "gmres"):
        cfg = RK.KrylovConfig(rel_tol=1e-8)
        r, nmv = RK.solve_trace_system(cond, b, cfg, solver)
        out[f"{solver}_x"] = r.x
        out[f"{solver}_iters"] = r.iterations
        out[f"{solver}_matvecs"] = nmv
        out[f"{solver}_converged"] = r.converged
        out[f"{solver}_history"] = np.array(r.history, dtype=float)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, out["fgmres_iters"], out["fgmres_matvecs"], out["gmres_iters"], out["gmres_matvecs"])


def dirk_case(name, case, n, m, p, dt, steps):
    import macrohdg.assembly as RA
    import macrohdg.stepper as RS
    from macrohdg.mesh import build_cube_mesh

    rd = RA.Discretization(build_cube_mesh(case.domain, n, m, periodic=(True,) * 3), p, case.params)
    f = rd.interpolate(case.initial_state)
    out = dict(versions=_versions(), n_ele=n, m=m, p=p, dt=dt, steps=steps, u0=f.u.copy(), q0=f.q.copy(),
               uhat0=f.uhat.copy())
    newton, kits, mvs, step_u, step_uhat, secs = [], [], [], [], [], []
    import time

    for _ in range(steps):
        t0 = time.perf_counter()
        sts, _dt = RS.dirk_advance(rd, f, dt, RS.DirkTableau.dirk33())
        secs.append(time.perf_counter() - t0)
        newton += [s.iterations for s in sts]
        kits += [s.krylov_iterations for s in sts]
        mvs += [s.krylov_matvecs for s in sts]
        step_u.append(f.u.copy())
        step_uhat.append(f.uhat.copy())
    out.update(u=f.u, q=f.q, uhat=f.uhat, newton=np.array(newton), krylov=np.array(kits), matvecs=np.array(mvs),
               step_u=np.stack(step_u), step_uhat=np.stack(step_uhat), seconds=np.array(secs))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, newton, kits, mvs)


def ptc_case(name, case, n, m, p, seed=0):
    import macrohdg.assembly as RA
    import macrohdg.stepper as RS
    from macrohdg.mesh import build_cube_mesh

    rd = RA.Discretization(build_cube_mesh(((0, 0, 0), (1, 1, 1)), n, m), p, case.params,
                           bcs=case.boundary_conditions(), source=case.source)
    f = rd.interpolate(case.exact_state)
    rng = np.random.default_rng(seed)
    f.u += rng.uniform(-1e-3, 1e-3, f.u.shape)
    f.uhat += rng.uniform(-1e-3, 1e-3, f.uhat.shape)
    f.q = rd.gradient_refresh(f.u, f.uhat)
    out = dict(versions=_versions(), n_ele=n, m=m, p=p, u0=f.u.copy(), q0=f.q.copy(), uhat0=f.uhat.copy())
    st, ptc = RS.ptc_steady_solve(rd, f, rel_tol=1e-10)
    out.update(u=f.u, q=f.q, uhat=f.uhat, newton=st.iterations, krylov=st.krylov_iterations,
               matvecs=st.krylov_matvecs, residuals=np.array(st.residuals), dtau=np.array(st.dtau))
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name, st.iterations, st.krylov_iterations, st.krylov_matvecs)


def tables_case(name):
    from macrohdg.basis import ref_macro
    from macrohdg.mesh import count_dofs_from_counts

    out = dict(versions=_versions())
    for m, p in [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (4, 1)]:
        rm = ref_macro(m, p)
        for k in ("sub_conn", "phi_vol", "grad_ref", "w_ref", "mass", "weak_deriv", "phi_face", "tri_conn",
                  "w_face_ref", "face_mass", "face_vol_nodes"):
            out[f"m{m}p{p}_{k}"] = getattr(rm, k)
    # DOF counts for the paper's Table 1 / Table 3 meshes (count_dofs, mesh.py:361-372)
    rows = []
    for nmac, nfac in [(768, 1632), (12, 30), (44, 108)]:
        for m, p in [(1, 3), (2, 3), (4, 3), (2, 4), (4, 2), (8, 1)]:
            rows.append((nmac, nfac, m, p) + count_dofs_from_counts(nmac, nfac, m, p))
    out["dof_rows"] = np.array(rows, dtype=np.int64)
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)
    print("wrote", name)


def main():
    sys.path.insert(0, REF)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    os.makedirs(OUT, exist_ok=True)
    from macrohdg.cases import CouetteCase, TgvCase

    tgv = TgvCase(reynolds=1600, mach=0.1)
    cou = CouetteCase()
    which = set(sys.argv[1:])

    def want(k):
        return not which or k in which

    if want("tables"):
        tables_case("tables")
    if want("op"):
        operator_case("op_tgv_m1p1", tgv, tgv.domain, 1, 1, 1, (True,) * 3, None, None, "dirk", True)
        operator_case("op_tgv_m2p2", tgv, tgv.domain, 1, 2, 2, (True,) * 3, None, None, "dirk", False)
        walls = {"y0": ("isothermal_noslip_wall", 1.0), "y1": ("isothermal_noslip_wall", 1.0)}
        operator_case("op_wall_m1p2", tgv, tgv.domain, 2, 1, 2, (True, False, True), walls, None, "ptc", False)
        operator_case("op_couette_m2p1", cou, ((0, 0, 0), (1, 1, 1)), 1, 2, 1, (False,) * 3,
                      cou.boundary_conditions(), cou.source, "ptc", True)
    if want("op23"):
        # n = L ns = 420 > 384: the larger-n batched LU path (C5 (m, p) = (2, 3))
        operator_case("op_tgv_m2p3", tgv, tgv.domain, 1, 2, 3, (True,) * 3, None, None, "dirk", False)
    if want("krylov"):
        krylov_case("krylov_tgv_m1p2", tgv, 1, 1, 2)
    if want("dirk"):
        dirk_case("dirk_tgv_m2p2", tgv, 1, 2, 2, 0.01, 1)
    if want("dirk48"):
        # a C3 slab: BASELINE configs[2]'s case, tableau, dt and (m, p) on 2^3 x 6 = 48 macros
        dirk_case("dirk_tgv_n2_m2p2", tgv, 2, 2, 2, 0.01, 2)
    if want("ptc"):
        ptc_case("ptc_couette_m2p1", cou, 1, 2, 1)


if __name__ == "__main__":
    main()
