"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per kernel class from an ncu
launch list (`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv`),
written to profiles/traffic.json for bench.py's roofline.traffic.

  python tools/traffic_from_ncu.py gpurun_out/traffic.csv profiles/traffic.json
"""
import collections
import csv
import json
import sys


def cls(n):
    if "gemm" in n:
        return "gemm"
    if "fwd_tc" in n:
        return "attn_fwd"
    if "dkdv" in n or "dq_tc" in n or "dq_tmem" in n or "bwd_dot" in n:
        return "attn_bwd"
    if "ce_rows" in n:
        return "ce_rows"
    if "rmsnorm" in n:
        return "rmsnorm"
    if n.startswith("void at::") or "at::native" in n:
        return None  # torch set-up kernels (synthetic data), not part of the step
    return "other"


rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
k, mn, mv, idc = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.defaultdict(dict)
for r in data:
    per[r[idc]][r[mn]] = float(r[mv].replace(",", ""))
    per[r[idc]]["name"] = r[k]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for d in per.values():
    c = cls(d["name"])
    if c is None:
        continue
    agg[c][0] += 1
    agg[c][1] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    agg[c][2] += d.get("gpu__time_duration.sum", 0)
out = {c: int(b / n) for c, (n, b, t) in agg.items()}
out["_source"] = ("ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum over warm-up + 1 L1 step "
                  "(tools/prof_step.py); mean DRAM bytes per launch per kernel class")
json.dump(out, open(sys.argv[2], "w"), indent=1)
print(json.dumps(out, indent=1))
