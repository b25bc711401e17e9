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
