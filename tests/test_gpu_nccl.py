"""The slab path over real NCCL (one process per GPU, tools/nccl_slab_check.py under
torchrun): the distributed apply and an FGMRES solve equal the single-process run.
Needs >= 2 GPUs; skips on one (the round's GPU box has one; tests/test_gpu_dist.py
covers the same code with thread ranks on one GPU, tests/test_dist_cpu.py with gloo)."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from gpu_util import need_gpu

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_nccl_slab_apply_and_solve(tmp_path):
    need_gpu()
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("needs >= 2 GPUs (one process per GPU over NCCL)")
    world = min(world, 4)
    subprocess.check_call([sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
                           "--nproc-per-node", str(world), os.path.join(ROOT, "tools", "nccl_slab_check.py"),
                           str(tmp_path)], timeout=900)
    for r in range(world):
        res = np.load(tmp_path / f"rank{r}.npy", allow_pickle=True).item()
        assert res["apply_equal"], (r, res)
        assert abs(res["iters"][0] - res["iters"][1]) <= 1, (r, res)
        assert res["x_err"] < 1e-8, (r, res)
