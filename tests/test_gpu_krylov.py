"""Fused device ICGS (mhdg_icgs) vs the reference formulation (krylov.py:51-58)
evaluated with torch in float64: same projections, norm and updated vector."""

import numpy as np
import pytest
import torch

from gpu_util import need_gpu
from paper_2402_11361_b200 import krylov as K

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,j", [(37, 0), (2080, 5), (2080, 59), (638976, 20)])
def test_fused_icgs_matches_reference_formulation(n, j):
    need_gpu()
    g = torch.Generator(device="cuda").manual_seed(n + j)
    V = torch.randn(61, n, dtype=torch.float64, device="cuda", generator=g)
    V[: j + 1] = torch.linalg.qr(V[: j + 1].T)[0].T  # orthonormal basis, as in Arnoldi
    w = torch.randn(n, dtype=torch.float64, device="cuda", generator=g) + 0.5 * V[0]
    Vj = V[: j + 1]
    h = Vj @ w
    wr = w - Vj.T @ h
    h2 = Vj @ wr
    wr = wr - Vj.T @ h2
    h_ref, hv_ref = (h + h2).cpu().numpy(), float(torch.linalg.vector_norm(wr))
    h_dev, hv_dev, w_dev = K._icgs_device(V, j, w)
    assert np.abs(h_dev - h_ref).max() <= 1e-12 * max(1.0, np.abs(h_ref).max())
    assert abs(hv_dev - hv_ref) <= 1e-12 * hv_ref
    assert float((w_dev - wr).abs().max()) <= 1e-12 * float(wr.abs().max())
    # deterministic
    h_b, hv_b, w_b = K._icgs_device(V, j, w)
    assert np.array_equal(h_b, h_dev) and hv_b == hv_dev and torch.equal(w_b, w_dev)
