"""Summarise an ncu SASS source page (csv) by regions between DMMA/BAR landmarks:
samples, instructions and stall reasons per region (for kernel tuning)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
data = rows[2:]
W = int(sys.argv[2]) if len(sys.argv) > 2 else 300
iS, iI, iSrc = hdr.index("# Samples"), hdr.index("Instructions Executed"), hdr.index("Source")
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {h: hdr.index(h) for h in stalls}
tot = sum(int(r[iS]) for r in data)
print("total samples", tot, "instructions", sum(int(r[iI]) for r in data))
for a in range(0, len(data), W):
    blk = data[a:a + W]
    s = sum(int(r[iS]) for r in blk)
    if s < 0.01 * tot:
        continue
    st = collections.Counter({h: sum(int(r[idx[h]] or 0) for r in blk) for h in stalls})
    ops = collections.Counter()
    for r in blk:
        t = r[iSrc].split()
        if t:
            op = t[1] if t[0].startswith("@") else t[0]
            ops[op.split(".")[0]] += 1
    print(f"[{a:5d}] {100 * s / tot:5.1f}% instr {sum(int(r[iI]) for r in blk):11d}  "
          + " ".join(f"{h[6:]}={100 * v / max(s, 1):.0f}%" for h, v in st.most_common(4))
          + f"  | DMMA {ops['DMMA']} BAR {ops['BAR']} LDS {ops['LDS']} LDG {ops['LDG']} STG {ops['STG']}")
