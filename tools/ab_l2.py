import os, sys
import torch
sys.path.insert(0, "/root/repo")
import bench
from paper_2402_11361_b200 import _lib
from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200 import condense as CD
L = _lib.lib()
case, disc = bench.c2_discretization(64)
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
CD.FACTOR = "lu"
lus = {}
for mode in (0, 2, 3, 4, 1, 2):
    L.mhdg_set_lu_l2mode(mode)
    cond = CD.CondensedSchur.allocate(blocks)
    st = disc.device.status_buffer()
    cond.refactor_async(st); torch.cuda.synchronize()
    with _lib.Timeline(64) as tl:
        for _ in range(3):
            cond.refactor_async(st)
        torch.cuda.synchronize()
    A.raise_status(st, "condense")
    print(f"mode {mode}: " + ", ".join(f"{k} {v / 3:.2f} ms" for k, v in tl.ms.items()), flush=True)
    lus[mode] = cond.lu.clone()
    del cond
print("equal:", all(torch.equal(lus[0], v) for v in lus.values()))
