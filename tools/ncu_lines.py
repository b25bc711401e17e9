"""Stall samples of an ncu report per CUDA source line: joins the SASS source page
(ncu -i X.ncu-rep --page source --csv) with nvdisasm -g line info of the object file,
instruction by instruction (same order).

    python tools/ncu_lines.py X.ncu-rep build/foo.o kernel_substring [min_pct]
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1:4]
minpct = float(sys.argv[4]) if len(sys.argv) > 4 else 0.5
raw = subprocess.check_output(["ncu", "-i", rep, "--page", "source", "--csv"], text=True, stderr=subprocess.DEVNULL)
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
iS, iI, iSrc = hdr.index("# Samples"), hdr.index("Instructions Executed"), hdr.index("Source")
iW, iWi = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
with tempfile.TemporaryDirectory() as td:
    subprocess.check_call(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=td, stdout=subprocess.DEVNULL)
    cub = [f for f in os.listdir(td) if f.endswith(".cubin")][0]
    sass = subprocess.check_output(["nvdisasm", "-g", "-c", os.path.join(td, cub)], text=True)
lines = []  # source line of each instruction of the kernel, in order
cur, infn = None, False
for ln in sass.splitlines():
    if ln.startswith(".text."):
        infn = kern in ln
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    if re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        lines.append(cur)
if len(lines) != len(data):
    print(f"warning: {len(lines)} disassembled instructions vs {len(data)} in the report", file=sys.stderr)
agg = collections.defaultdict(lambda: collections.Counter())
for r, l in zip(data, lines):
    a = agg[l]
    a["samples"] += int(r[iS] or 0)
    a["inst"] += int(r[iI] or 0)
    a["shw"] += int(r[iW] or 0)
    a["shwi"] += int(r[iWi] or 0)
    for h in stalls:
        a[h] += int(r[hdr.index(h)] or 0)
tot = sum(a["samples"] for a in agg.values())
toti = sum(a["inst"] for a in agg.values())
print(f"total samples {tot}, warp instructions {toti}")
src = {}
for l, a in sorted(agg.items(), key=lambda kv: (kv[0] or ("", 0))):
    if a["samples"] < minpct / 100 * tot:
        continue
    f, n = l if l else ("?", 0)
    if f not in src:
        p = os.path.join(os.path.dirname(os.path.abspath(obj)), "..", f)
        src[f] = open(p).read().splitlines() if os.path.exists(p) else []
    text = src[f][n - 1].strip() if 0 < n <= len(src[f]) else ""
    st = " ".join(f"{h[6:]}={100 * a[h] / max(a['samples'], 1):.0f}%" for h in sorted(stalls, key=lambda h: -a[h])[:3])
    print(f"{f}:{n:4d} {100 * a['samples'] / tot:5.1f}% inst {100 * a['inst'] / toti:5.1f}% smem wavefronts "
          f"{a['shw']:>10d}/{a['shwi']:<10d} {st} | {text[:100]}")
