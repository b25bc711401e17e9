import sys, os, json, time
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import numpy as np, torch
from test_gpu_krylov import _c1_operator
from paper_2402_11361_b200 import _lib
L = _lib.lib()
d, cond = _c1_operator()
x = torch.randn(d.n_trace, dtype=torch.float64, device="cuda")
ref = cond.apply_trace(x).clone()
def gtime(fn, reps=300):
    fn(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.capture_begin(); out = fn(); g.capture_end()
    torch.cuda.current_stream().wait_stream(s)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    return round(1e3 * e0.elapsed_time(e1) / reps, 2), out
res = {}
for name, setup in [("split", lambda: (L.mhdg_set_stream_enabled(1), L.mhdg_set_apply_split(1))),
                    ("generic", lambda: (L.mhdg_set_stream_enabled(0), L.mhdg_set_apply_split(1)))]:
    setup()
    t, out = gtime(lambda: cond.apply_trace(x))
    res[name] = t
    res[name + "_maxdiff"] = float((out - ref).abs().max() / ref.abs().max())
L.mhdg_set_stream_enabled(1)
print(json.dumps(res))
