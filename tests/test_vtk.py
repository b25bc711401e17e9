"""Legacy VTK writer (the reference's missing io_utils.write_vtk, mesh.py:375-379):
cell counts, corner lattice nodes, and point data round-trip.  CPU only."""

import numpy as np

from golden_cases import TGV
from paper_2402_11361_b200.cases import UniformFlow2D
from paper_2402_11361_b200.discretization import Discretization
from paper_2402_11361_b200.mesh import build_cube_mesh, build_square_mesh
from paper_2402_11361_b200.vtk import _corner_nodes, primitives, write_vtk


def _read(path):
    lines = open(path).read().split("\n")
    head = {ln.split()[0]: ln for ln in lines if ln and ln.split()[0] in ("POINTS", "CELLS", "CELL_TYPES", "POINT_DATA")}
    return lines, head


def test_vtk_3d_and_2d(tmp_path):
    d3 = Discretization(build_cube_mesh(TGV.domain, 1, 2, periodic=(True,) * 3), 2, TGV.params)
    u, _ = d3.nodal_interpolant(TGV.initial_state)
    write_vtk(d3, tmp_path / "tgv.vtk", u)
    lines, head = _read(tmp_path / "tgv.vtk")
    assert head["POINTS"].split()[1] == str(d3.n_mac * d3.L)
    assert head["CELLS"].split()[1] == str(d3.n_mac * d3.rm.n_sub)
    # sub-element corners are lattice nodes at the sub-element vertices
    c = _corner_nodes(d3.rm)
    assert c.shape == (8, 4) and len(np.unique(c)) == 10  # m=2: 4 corners + 6 edge midpoints
    i = lines.index("SCALARS rho double 1") + 2
    rho = np.array([float(v) for v in lines[i: i + d3.n_mac * d3.L]])
    assert np.allclose(rho, primitives(u, d3.params.gamma)[0].reshape(-1))
    c2 = UniformFlow2D()
    d2 = Discretization(build_square_mesh(c2.domain, 2, 4, periodic=(True, True)), 3, c2.params)
    write_vtk(d2, tmp_path / "c2.vtk")
    _, head2 = _read(tmp_path / "c2.vtk")
    assert head2["CELLS"].split()[1] == str(d2.n_mac * 16)
    assert "POINT_DATA" not in head2
