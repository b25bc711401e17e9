"""Pin the CPU oracle (oracle/) and the host setup against reference outputs.

The fixtures in tests/golden were produced by running the reference itself
(oracle/make_golden.py).  CPU only."""

import numpy as np
import pytest

import oracle.hdg_oracle as O
from conftest import load_golden, rel_err
from golden_cases import COU, OP_CASES, TGV, ctx_of
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_cube_mesh, count_dofs_from_counts
from paper_2402_11361_b200.refmacro import ref_macro

TOL = 1e-12


def test_reference_tables():
    g = load_golden("tables")
    for key, val in g.items():
        if not key.startswith("m"):
            continue
        mp, name = key.split("_", 1)
        m, p = int(mp[1]), int(mp[3])
        mine = getattr(ref_macro(3, m, p), name)
        assert mine.shape == val.shape, key
        assert np.max(np.abs(mine - val)) < 1e-12 * max(1.0, np.max(np.abs(val))), key


def test_dof_counts_table():
    g = load_golden("tables")
    for nm, nf, m, p, tot, tr, per in g["dof_rows"]:
        assert count_dofs_from_counts(int(nm), int(nf), int(m), int(p), 5, 3) == (tot, tr, per)


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_layout_matches_reference(name):
    g = load_golden(name)
    d = OP_CASES[name]()
    assert np.array_equal(d.gather, g["gather"])
    assert np.array_equal(d.mesh.face_macros, g["face_macros"])
    assert np.array_equal(d.mesh.corner_map, g["corner_map"])
    for k in ("normals", "areas", "det", "h_sub"):
        assert rel_err(getattr(d, k), g[k]) < 1e-14


@pytest.mark.parametrize("name", sorted(OP_CASES))
def test_oracle_operator_vs_reference(name):
    g = load_golden(name)
    d = OP_CASES[name]()
    f = O.Fields(g["u"], g["q"], g["uhat"])
    ctx = ctx_of(g, O.Ctx)
    res = O.residual(d, f, ctx)
    # R_Q cancels to O(1e-3) of its terms; compare against its own term scale
    assert np.max(np.abs(res[0] - g["R_Q"])) < 1e-12 * np.max(np.abs(O.grad_mass_apply(d, f.q)))
    assert rel_err(res[1], g["R_U"]) < TOL
    assert rel_err(res[2], g["R_T"]) < 1e-11
    blocks, frozen = O.jacobian(d, f, ctx)
    for k in ("state_state", "face_state_trace", "face_trace_state", "face_trace_trace", "wdgdq_vol",
              "wdgdq_face", "trace_face_scale"):
        arr = getattr(blocks, k)
        ref = g[f"blk_{k}"]
        assert rel_err(arr[: len(ref)], ref) < TOL, k
        assert rel_err(arr.reshape(len(arr), -1).sum(1), g[f"sum_{k}"]) < 1e-11, k
    assert rel_err(frozen.supg_tau, g["frz_supg_tau"]) < TOL
    cond = O.condense(blocks)
    S = O.schur_matrix(blocks)
    assert rel_err(np.einsum("mab,mb->ma", S, g["schur_probe"]), g["schur_times_probe"]) < TOL
    assert rel_err(cond.schur_solve(g["schur_probe"]), g["schur_inv_times_probe"]) < 1e-10
    for x, y in zip(g["x"], g["y"]):
        assert rel_err(cond.apply_trace(x), y) < 1e-11
    assert rel_err(cond.rhs(*res), g["rhs"]) < 1e-10
    du, dq = cond.recover(res[0], res[1], g["x"][0])
    assert rel_err(du, g["rec_du"]) < 1e-10
    assert rel_err(dq, g["rec_dq"]) < 1e-10
    pre = O.block_precond_build(cond)
    assert rel_err(pre(g["x"][0]), g["precond_y"]) < 1e-11
    if "dense_A" in g:
        A = O.dense_trace_operator(blocks)
        assert rel_err(A, g["dense_A"]) < 1e-10
        assert rel_err(A @ g["x"][1], g["y"][1]) < 1e-11


def test_oracle_krylov_vs_reference():
    g = load_golden("krylov_tgv_m1p2")
    d = Discretization(build_cube_mesh(TGV.domain, 1, 1, periodic=(True,) * 3), 2, TGV.params)
    f = O.Fields(g["u"], g["q"], g["uhat"])
    ctx = O.Ctx(50.0, g["hist"], np.inf, 0.02)
    res = O.residual(d, f, ctx)
    blocks, _ = O.jacobian(d, f, ctx)
    cond = O.condense(blocks)
    b = cond.rhs(*res)
    assert rel_err(b, g["rhs"]) < 1e-10
    for solver in ("fgmres", "gmres"):
        r, nmv = O.solve_trace_system(cond, b, O.KrylovConfig(rel_tol=1e-8), solver)
        assert r.iterations == int(g[f"{solver}_iters"])
        assert nmv == int(g[f"{solver}_matvecs"])
        assert rel_err(r.x, g[f"{solver}_x"]) < 1e-8


def test_oracle_dirk_step_vs_reference():
    g = load_golden("dirk_tgv_m2p2")
    d = Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 2, TGV.params)
    f = O.Fields(g["u0"].copy(), g["q0"].copy(), g["uhat0"].copy())
    sts, _ = O.dirk_advance(d, f, float(g["dt"]), O.DirkTableau.dirk33())
    assert [s.iterations for s in sts] == list(g["newton"])
    assert [s.krylov_iterations for s in sts] == list(g["krylov"])
    assert [s.krylov_matvecs for s in sts] == list(g["matvecs"])
    assert rel_err(f.u, g["u"]) < 1e-8
    assert rel_err(f.uhat, g["uhat"]) < 1e-8


@pytest.mark.slow
def test_oracle_ptc_couette_vs_reference():
    g = load_golden("ptc_couette_m2p1")
    d = Discretization(build_cube_mesh(((0, 0, 0), (1, 1, 1)), 1, 2), 1, COU.params,
                       bcs=COU.boundary_conditions(), source=COU.source)
    f = O.Fields(g["u0"].copy(), g["q0"].copy(), g["uhat0"].copy())
    st, _ = O.ptc_steady_solve(d, f, rel_tol=1e-10)
    assert abs(st.iterations - int(g["newton"])) <= 1
    assert abs(st.krylov_iterations - int(g["krylov"])) <= 1
    assert rel_err(f.u, g["u"]) < 1e-8
    assert rel_err(f.uhat, g["uhat"]) < 1e-8
