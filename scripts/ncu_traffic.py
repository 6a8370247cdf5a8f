"""Per-launch DRAM traffic of the bench step's kernels from one ncu capture.

Runs on the GPU box:
  ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      -k regex:"k_(jac|side|vanka)" --csv python scripts/prof_step.py cfg2 3 > gpurun_out/traffic.csv
then here:  python scripts/ncu_traffic.py gpurun_out/traffic.csv profiles/traffic_r01.json
"""
import csv
import json
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
iK, iN, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
per = defaultdict(lambda: defaultdict(list))
for r in rows[1:]:
    k = r[iK]
    name = ("k_jacobian" if "k_jacobian" in k else "k_jac_post" if "k_jac_post" in k else
            "k_side_products" if "k_side_products" in k else
            "k_vanka_gemv" if "gemv" in k else
            "k_vanka_scatter" if "scatter" in k else k[:40])
    per[name][r[iN]].append(float(r[iV].replace(",", "")))
out = {}
for name, m in per.items():
    n = len(m["gpu__time_duration.sum"])
    rd = sum(m["dram__bytes_read.sum"]) / n
    wr = sum(m["dram__bytes_write.sum"]) / n
    out[name] = {"launches": n, "dram_bytes_per_launch": rd + wr, "read": rd, "write": wr,
                 "ns_per_launch": sum(m["gpu__time_duration.sum"]) / n}
res = {"kernels": out,
       "jacobian_apply": sum(out[k]["dram_bytes_per_launch"] for k in ("k_jacobian", "k_side_products", "k_jac_post")
                             if k in out),
       "vanka_gemv": out.get("k_vanka_gemv", {}).get("dram_bytes_per_launch"),
       "vanka_scatter": out.get("k_vanka_scatter", {}).get("dram_bytes_per_launch"),
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (cold caches, serialized) on "
                 + (sys.argv[3] if len(sys.argv) > 3 else "scripts/prof_step.py cfg2 3")}
json.dump(res, open(sys.argv[2], "w"), indent=1)
print(json.dumps(res, indent=1))
