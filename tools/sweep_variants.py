"""Time the C2 apply with each libmhdg variant given on the command line
(tools/build_variants.sh) and check it against the generic kernel."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import ctypes as C, sys, torch
sys.path.insert(0, ROOT)
from paper_2402_11361_b200 import _lib
_lib.LIB_PATH = SO
import bench
from paper_2402_11361_b200 import assembly as A
from paper_2402_11361_b200.condense import CondensedSchur
L = _lib.lib()
case, disc = bench.c2_discretization()
u, uhat = bench.c2_state(case, disc)
f = A.FieldState(torch.as_tensor(u, device="cuda"), None, torch.as_tensor(uhat, device="cuda"))
f.q = A.gradient_refresh(disc, f.u, f.uhat)
blocks, _ = A.jacobian(disc, f, A.StageContext.steady(1.0))
cond = CondensedSchur.build(blocks)
xs = torch.randn(22, disc.n_trace, dtype=torch.float64, device="cuda")
L.mhdg_set_stream_enabled(0)
ref = cond.apply_trace(xs[0]).clone()
L.mhdg_set_stream_enabled(1)
got = cond.apply_trace(xs[0]).clone()
err = float((got - ref).abs().max() / ref.abs().max())
for i in range(2):
    cond.apply_trace(xs[i])
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(20):
    cond.apply_trace(xs[2 + i])
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
b = bench.algorithmic_bytes_per_macro(disc) * disc.n_mac
L.mhdg_stream_grid.restype = C.c_int
print(f"{os.path.basename(SO):18s} grid {L.mhdg_stream_grid():4d}  {ms:.3f} ms  {b / ms / 1e6:.0f} GB/s  err {err:.1e}")
'''

for so in sys.argv[1:]:
    code = "import os\nROOT=%r\nSO=%r\n" % (ROOT, os.path.abspath(so)) + CHILD
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    print(r.stdout.strip() or r.stderr.strip()[-800:], flush=True)
