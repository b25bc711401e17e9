"""Diagnostic: couplings-only blocks from k_couplings vs k_assemble (want_jac = 2), per array."""
import os, sys
import numpy as np
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2402_11361_b200 import _lib, assembly as A
import test_gpu_recompute as T

for name, mk in (("c2", T._c2_patch), ("tgv", T._tgv), ("tgv6", lambda: T._tgv(6))):
    disc, f, ctx = mk()
    rb = A.RecomputeBlocks(disc, f, ctx, chunk=disc.n_mac)
    wins = []
    for knob in (1, 0):
        _lib.lib().mhdg_set_couplings_kernel(knob)
        w = A.LocalBlocks.empty(disc, with_state_state=False)
        for k in w.KEYS:
            if k != "state_state":
                getattr(w, k).fill_(float("nan"))
        rb.assemble_window(0, disc.n_mac, 2, w, None)
        torch.cuda.synchronize()
        wins.append(w)
    full, _ = A.jacobian(disc, f, ctx, recompute=False)
    for k in w.KEYS:
        if k == "state_state":
            continue
        a, b, c = getattr(wins[0], k), getattr(wins[1], k), getattr(full, k)
        ne = (a != b) & ~(torch.isnan(a) & torch.isnan(b))
        print(name, k, "kernel-vs-asm2 mismatches", int(ne.sum()), "of", a.numel(), "nan", int(torch.isnan(a).sum()),
              "max abs diff", float((a - b).abs().nan_to_num().max()), "asm2-vs-full", int((b != c).sum()))
        if ne.any():
            ns = disc.ns
            if a.dim() == 4 and a.shape[-1] == a.shape[-2]:
                nz = ne.nonzero()
                st = {}
                for r, c in zip((nz[:, 2] % ns).tolist(), (nz[:, 3] % ns).tolist()):
                    st[(r, c)] = st.get((r, c), 0) + 1
                print("    (s,t) histogram", st, "macros", sorted(set(nz[:, 0].tolist()))[:10])
            idx = ne.nonzero()[:5]
            for i in idx:
                t = tuple(int(v) for v in i)
                print("   ", t, float(a[t]), float(b[t]))
