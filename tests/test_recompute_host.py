"""Host logic of the coupling-recompute representation (no GPU): jacobian() dispatch,
the linearisation snapshot, the window size rules and the window partition."""

from types import SimpleNamespace

import torch

from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200.cases import UniformFlow2D
from paper_2402_11361_b200.condense import CondensedRecompute


def _fake(n_mac=10):
    disc = SimpleNamespace(n_mac=n_mac, params=UniformFlow2D().params, device=None, is_distributed=False)
    f = A.FieldState(torch.zeros((n_mac, 3, 4), dtype=torch.float64), torch.zeros((n_mac, 2, 3, 4), dtype=torch.float64),
                     torch.zeros(7, dtype=torch.float64))
    return disc, f


def test_jacobian_returns_the_linearisation_point(monkeypatch):
    disc, f = _fake()
    blocks, frozen = A.jacobian(disc, f, A.StageContext.steady(1.0), recompute=True)
    assert isinstance(blocks, A.RecomputeBlocks) and frozen is None
    f.u += 1.0  # the caller moves on; the condensation keeps its own copy
    assert float(blocks.u.abs().max()) == 0.0
    assert blocks.stage.pseudo_dt == 1.0 and blocks.stage.hist is None
    monkeypatch.setenv("MHDG_APPLY_REPR", "recompute")
    blocks2, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
    assert isinstance(blocks2, A.RecomputeBlocks)


def test_window_size_and_partition(monkeypatch):
    disc, f = _fake(10)
    ctx = A.StageContext.steady()
    assert A.RecomputeBlocks(disc, f, ctx, chunk=4).chunk == 4
    assert A.RecomputeBlocks(disc, f, ctx, chunk=64).chunk == 10  # never more than the mesh
    assert A.RecomputeBlocks(disc, f, ctx).chunk == 10  # default 4096, clamped
    monkeypatch.setenv("MHDG_RECOMPUTE_CHUNK", "3")
    rb = A.RecomputeBlocks(disc, f, ctx)
    assert rb.chunk == 3
    wins = CondensedRecompute._windows(SimpleNamespace(disc=disc, blocks=rb))
    assert wins == [(0, 3), (3, 3), (6, 3), (9, 1)]
    assert sum(c for _, c in wins) == disc.n_mac
