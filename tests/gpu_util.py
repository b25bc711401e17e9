"""Helpers shared by the GPU parity tests."""

import numpy as np
import pytest
import torch

import oracle.hdg_oracle as O
from paper_2402_11361_b200.assembly import LocalBlocks


def need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def dev(a):
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


def upload_blocks(disc, ob):
    return LocalBlocks.from_arrays(disc, {k: getattr(ob, k) for k in LocalBlocks.KEYS})


def perturbed_fields(disc, state_fn, seed, amp_u=1e-3, amp_q=1e-2):
    f = O.interpolate(disc, state_fn)
    rng = np.random.default_rng(seed)
    f.u = f.u + amp_u * rng.standard_normal(f.u.shape) * np.abs(f.u).max()
    f.uhat = f.uhat + amp_u * rng.standard_normal(f.uhat.shape) * np.abs(f.uhat).max()
    f.q = f.q + amp_q * rng.standard_normal(f.q.shape)
    return f


def subset_disc(disc, idx):
    """A host Discretization restricted to the macros `idx` (sorted), sharing the
    global trace numbering: the oracle run on it reproduces exactly those macros'
    local operators (every per-macro array is sliced; gather still indexes the
    full trace vector, so a global x gathers the same local traces)."""
    import copy

    sub = copy.copy(disc)
    idx = np.asarray(idx)
    sub.n_mac = len(idx)
    for k in ("det", "inv_jac", "jac", "origin", "normals", "areas", "h_sub", "gather", "bc_kind", "bc_label"):
        setattr(sub, k, getattr(disc, k)[idx])
    sub._device = None
    return sub
