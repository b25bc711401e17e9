"""Rebuild the discretizations the golden fixtures were generated on."""

import numpy as np

from paper_2402_11361_b200.cases import CouetteCase, TgvCase
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_cube_mesh

TGV = TgvCase(reynolds=1600, mach=0.1)
COU = CouetteCase()
WALLS = {"y0": ("isothermal_noslip_wall", 1.0), "y1": ("isothermal_noslip_wall", 1.0)}

OP_CASES = {
    "op_tgv_m1p1": lambda: Discretization(build_cube_mesh(TGV.domain, 1, 1, periodic=(True,) * 3), 1, TGV.params),
    "op_tgv_m2p2": lambda: Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 2, TGV.params),
    "op_tgv_m2p3": lambda: Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 3, TGV.params),
    "op_wall_m1p2": lambda: Discretization(build_cube_mesh(TGV.domain, 2, 1, periodic=(True, False, True)), 2,
                                           TGV.params, bcs=WALLS),
    "op_couette_m2p1": lambda: Discretization(build_cube_mesh(((0, 0, 0), (1, 1, 1)), 1, 2), 1, COU.params,
                                              bcs=COU.boundary_conditions(), source=COU.source),
}


def ctx_of(g, ctx_cls):
    if str(g["ctx_kind"]) == "dirk":
        return ctx_cls(float(g["dt_coeff"]), g["hist"], float(g["pseudo_dt"]), float(g["supg_dt"]))
    return ctx_cls(0.0, None, float(g["pseudo_dt"]), float(g["supg_dt"]))
