"""Per-kernel mean duration / DRAM bytes from an ncu --csv launch list."""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
i = next(k for k, r in enumerate(rows) if r and r[0] == "ID")
h = rows[i]
iK, iM, iV = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
acc = defaultdict(lambda: defaultdict(list))
for r in rows[i + 1:]:
    if len(r) > iV:
        acc[r[iK].split("(")[0][-40:]][r[iM]].append(float(r[iV].replace(",", "")))
for k, m in acc.items():
    t = m.get("gpu__time_duration.sum", [0])
    rd = m.get("dram__bytes_read.sum", [0]); wr = m.get("dram__bytes_write.sum", [0])
    print(f"{k:42s} n={len(t):3d} t={sum(t)/len(t)/1e3:8.1f}us  rd={sum(rd)/len(rd)/1e6:8.2f}MB wr={sum(wr)/len(wr)/1e6:7.2f}MB")
