"""profiles/traffic.json from an ncu launch list (gpu__time_duration, dram__bytes_read/write per launch):
mean DRAM bytes per launch of each library kernel, keyed like bench.py's timeline slots."""
import collections
import csv
import json
import sys

src, out = sys.argv[1], sys.argv[2]
rows = list(csv.reader(open(src)))
start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[start]
rows = [r for r in rows[start + 1:] if len(r) == len(h)]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
per = collections.defaultdict(dict)
for r in rows:
    per[(int(r[ii]), r[ki])][r[mi]] = float(r[vi].replace(",", ""))


def slot(name):
    if "k_apply_stream" in name:
        part = name.split(">,")[1].split(">")[0].split(",")[-1].strip()  # <Cfg<..>, STAGES, PART>
        return {"1": "apply_pre", "2": "apply_post", "0": "apply_fused"}.get(part)
    for pat, key in (("k_lu_warp", "apply_si"), ("k_si_stream", "apply_si"), ("k_schur2", "schur"),
                     ("k_schur_mma", "schur"), ("k_pack_lu4", "pack"), ("k_pack_inv_rows", "pack"),
                     ("k_lu4", "factor"), ("k_gj3", "factor"), ("k_face_reduce", "face_reduce"),
                     ("k_ahat_gemv", "apply_ahat")):
        if pat in name:
            return key
    return None


acc = collections.defaultdict(list)
for (i, name), m in per.items():
    k = slot(name)
    if k and "dram__bytes_read.sum" in m:
        acc[k].append(m["dram__bytes_read.sum"] + m.get("dram__bytes_write.sum", 0.0))
res = {"source": f"{src}: ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                 "--clock-control none, python bench.py --steps 2 --warmup 3 (C2), mean over launches"}
for k, v in sorted(acc.items()):
    res[k + "_dram_bytes_per_launch"] = int(sum(v) / len(v))
if all(k in acc for k in ("apply_pre", "apply_si", "apply_post")):
    res["apply_local_dram_bytes_per_launch"] = sum(res[k + "_dram_bytes_per_launch"]
                                                   for k in ("apply_pre", "apply_si", "apply_post"))
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
