"""C4 (flow past a sphere): the O-grid mesher with its pole wedges, the adiabatic
no-slip wall, and GPU parity with the oracle restatement.  The reference can run
neither (box meshes only, no adiabatic wall), so the new wall rows
are pinned by central finite differences of the oracle residual and the device
path by the oracle (itself pinned to the reference in 3D)."""

import numpy as np
import pytest

import oracle.hdg_oracle as O
from conftest import load_golden, rel_err
from oracle.make_sphere_golden import NEWTON_STEPS, sphere_setup
from paper_2402_11361_b200.cases import SphereCase
from paper_2402_11361_b200.discretization import ADIABATIC, DIRICHLET, Discretization
from paper_2402_11361_b200.mesh import BOUNDARY, BOUNDARY_LABELS, INTERIOR, build_sphere_ogrid_mesh, count_dofs


def test_ogrid_mesh_structure():
    n_r, n_t, n_p = 3, 4, 6
    m = build_sphere_ogrid_mesh(n_r, n_t, n_p, 2, r_in=0.5, r_out=4.0)
    # every cell gives 6 Kuhn tets except the polar wedges, which keep 3
    assert m.n_macro == 6 * n_r * n_t * n_p - 3 * n_r * 2 * n_p
    assert np.all(m.det > 0)
    # conforming: every face is interior (two sides) or on one of the two spheres
    kinds = m.face_kind
    assert set(np.unique(kinds)) <= {INTERIOR, BOUNDARY}
    assert np.all(m.face_macros[kinds == INTERIOR, 1] >= 0)
    labels = m.face_label[kinds == BOUNDARY]
    assert set(np.unique(labels)) == {BOUNDARY_LABELS.index("sphere"), BOUNDARY_LABELS.index("farfield")}
    # each sphere is tiled: 2 triangles per quad cell face, 1 per polar wedge face
    n_b = 2 * (n_t - 2) * n_p + 2 * n_p
    assert np.sum(labels == BOUNDARY_LABELS.index("sphere")) == n_b
    assert np.sum(labels == BOUNDARY_LABELS.index("farfield")) == n_b
    # boundary vertices lie on their spheres; boundary face normals point out of the shell
    for lbl, rad, sgn in (("sphere", 0.5, -1.0), ("farfield", 4.0, 1.0)):
        sel = np.nonzero((kinds == BOUNDARY) & (m.face_label == BOUNDARY_LABELS.index(lbl)))[0]
        mac, lf = m.face_macros[sel, 0], m.face_locals[sel, 0]
        keep = lf[:, None] != np.arange(4)[None, :]
        verts = m.vertices[m.macro_tets[mac][keep].reshape(-1, 3)]
        assert np.allclose(np.linalg.norm(verts, axis=-1), rad)
        centroid = m.vertices[m.macro_tets[mac]].mean(axis=1)
        assert np.all(sgn * np.einsum("fk,fk->f", m.normals[mac, lf], centroid) > 0)
    # the tets fill the polyhedral shell: volume approaches the spherical shell's
    vols = [build_sphere_ogrid_mesh(3, k, 2 * k, 1, r_in=0.5, r_out=4.0).macro_volumes().sum() for k in (4, 8, 16)]
    exact = 4.0 / 3.0 * np.pi * (4.0**3 - 0.5**3)
    errs = [abs(v - exact) / exact for v in vols]
    assert errs[0] > errs[1] > errs[2] and errs[2] < 0.03
    # r-major cell order: macro slabs are radial shells
    rv = np.round(np.linalg.norm(m.vertices, axis=1), 12)
    shell = np.searchsorted(np.unique(rv), rv)[m.macro_tets].min(axis=1)
    assert np.all(np.diff(shell) >= 0) and shell[-1] == n_r - 1


def test_ogrid_full_c4_counts():
    """BASELINE configs[3] mesh: 32 x 24 x 48 cells (grading 1.15, r = 0.5 .. 20)."""
    m = build_sphere_ogrid_mesh(32, 24, 48, 2)
    assert m.n_macro == 221184 - 32 * 2 * 48 * 3  # 211,968 after the pole wedges
    assert np.all(m.det > 0)
    r = np.unique(np.round(np.linalg.norm(m.vertices, axis=1), 10))
    assert abs(r[0] - 0.5) < 1e-12 and abs(r[-1] - 20.0) < 1e-9
    dr = np.diff(r)
    assert np.allclose(dr[1:] / dr[:-1], 1.15)
    tot, tr, per = count_dofs(m, 2)
    assert per == 5 * 4 * 35 and tr == 5 * m.n_faces * 15


def _small(p=2, m=1):
    c = SphereCase()
    d = Discretization(build_sphere_ogrid_mesh(2, 3, 4, m, r_out=3.0), p, c.params, bcs=c.boundary_conditions())
    return c, d


def test_adiabatic_wall_rows():
    c, d = _small()
    kinds = {k for k, _ in d.bc_data.values()}
    assert kinds == {ADIABATIC, DIRICHLET}
    f = O.interpolate(d, c.freestream)
    res = O.residual(d, f, O.Ctx.steady())
    # at the free stream only the wall rows (m_hat = 0) are violated
    wall = d.bc_kind == ADIABATIC
    R_T = res[2].reshape(-1, d.Lf, d.ns)
    f_wall = np.unique(d.mesh.faces_of_macro[wall])
    others = np.setdiff1d(np.arange(d.mesh.n_faces), f_wall)
    assert np.max(np.abs(R_T[others])) < 1e-12 * np.max(np.abs(f.u))
    assert np.max(np.abs(R_T[f_wall][..., 1])) > 1e-3  # x-momentum trace against m_hat = 0
    assert np.max(np.abs(R_T[f_wall][..., [0, 2, 3, 4]])) < 1e-12 * np.max(np.abs(f.u))


def _fd(fun, eps):
    return (fun(eps) - fun(-eps)) / (2 * eps)


def test_adiabatic_wall_jacobian_finite_differences():
    c, d = _small()
    f = O.interpolate(d, c.freestream)
    rng = np.random.default_rng(4)
    f.u = f.u * (1.0 + 1e-3 * rng.standard_normal(f.u.shape))
    f.uhat = f.uhat * (1.0 + 1e-3 * rng.standard_normal(f.uhat.shape))
    ctx = O.Ctx(5.0, -0.2 * f.u, np.inf, 0.05)
    blocks, frozen = O.jacobian(d, f, ctx)
    M = d.n_mac

    def R(u, q, uh):
        return O.residual(d, O.Fields(u, q, uh), ctx, frozen=frozen)

    du = rng.standard_normal(f.u.shape) * np.abs(f.u).max() * 1e-2
    dq = rng.standard_normal(f.q.shape) * 1e-2
    dh = rng.standard_normal(f.uhat.shape) * np.abs(f.uhat).max() * 1e-2
    fdU = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u + s * du, f.q, f.uhat)[1:]]), 1e-4)
    jU = np.einsum("mab,mb->ma", blocks.state_state, du.reshape(M, -1)).ravel()
    n_u = jU.size
    assert rel_err(jU, fdU[:n_u]) < 1e-6
    assert rel_err(O.scatter_add(d, O.trace_state_apply(blocks, du)), fdU[n_u:]) < 1e-6
    fdQ = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u, f.q + s * dq, f.uhat)[1:]]), 1e-4)
    assert rel_err(O.state_grad_apply(blocks, dq).ravel(), fdQ[:n_u]) < 1e-6
    assert rel_err(O.scatter_add(d, O.trace_grad_apply(blocks, dq)), fdQ[n_u:]) < 1e-6
    fdH = _fd(lambda s: np.concatenate([r.ravel() for r in R(f.u, f.q, f.uhat + s * dh)[1:]]), 1e-4)
    xl = O.gather_local(d, dh)
    assert rel_err(O.state_trace_apply(blocks, xl).ravel(), fdH[:n_u]) < 1e-6
    assert rel_err(O.scatter_add(d, O.trace_trace_apply(blocks, xl)), fdH[n_u:]) < 1e-6
    # condensed operator == dense one-shot elimination; the wall-face preconditioner blocks are SPD
    cond = O.condense(blocks)
    A = O.dense_trace_operator(blocks)
    x = rng.standard_normal(d.n_trace)
    assert rel_err(cond.apply_trace(x), A @ x) < 1e-11
    O.block_precond_build(cond)


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_sphere_assembly_and_apply_vs_oracle():
    from gpu_util import dev, host, need_gpu, perturbed_fields
    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200.condense import condense

    need_gpu()
    for p, m in ((2, 1), (1, 2), (2, 2)):
        c, d = _small(p, m)
        of = perturbed_fields(d, c.freestream, 7)
        f = A.to_device_fields(d, of.u, of.q, of.uhat)
        octx, gctx = O.Ctx.steady(2.0), A.StageContext.steady(2.0)
        (oq, ou, ot), ob, _ = O.assemble_system(d, of, octx)
        (gq, gu, gt), gb, _ = A.assemble_system(d, f, gctx)
        assert rel_err(host(gu), ou) < 1e-10
        assert rel_err(host(gt), ot) < 1e-10
        for k in ("state_state", "face_state_trace", "face_trace_state", "face_trace_trace", "wdgdq_vol",
                  "wdgdq_face", "trace_face_scale"):
            assert rel_err(host(getattr(gb, k)), getattr(ob, k)) < 1e-10, (p, m, k)
        ocond, gcond = O.condense(ob), condense(gb)
        x = np.random.default_rng(3).standard_normal(d.n_trace)
        assert rel_err(host(gcond.apply_trace(dev(x))), ocond.apply_trace(x)) < 1e-9, (p, m)
        assert rel_err(host(gcond.rhs(gq, gu, gt)), ocond.rhs(oq, ou, ot)) < 1e-9, (p, m)


@pytest.mark.gpu
def test_sphere_ptc_newton_vs_oracle():
    """The C4 workload (5 PTC Newton steps from the perturbed free stream) at test
    size: residual history, pseudo-time steps and Krylov counts against the oracle."""
    from gpu_util import host, need_gpu
    from paper_2402_11361_b200 import assembly as A
    from paper_2402_11361_b200 import stepper as S

    need_gpu()
    g = load_golden("sphere_ptc_oracle")
    _, d, _, _ = sphere_setup()
    f = A.to_device_fields(d, g["u0"], g["q0"], g["uhat0"])
    ptc = S.PtcState(dtau=1.0, tau_init=1.0, tau_max=1e8)
    st = S.newton_solve(d, f, A.StageContext.steady(), max_newton=NEWTON_STEPS, ptc=ptc, abs_tol=1e-10,
                        rel_tol=1e-10)
    assert st.iterations == int(g["newton"])
    assert abs(st.krylov_iterations - int(g["krylov"])) <= NEWTON_STEPS
    assert np.allclose(st.residuals, g["residuals"], rtol=1e-6)
    assert rel_err(host(f.u), g["u"]) < 1e-7
    assert rel_err(host(f.uhat), g["uhat"]) < 1e-7
