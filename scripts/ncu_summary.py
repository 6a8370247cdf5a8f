"""Summarise an ncu report of one kernel: headline metrics, stall reasons,
instruction mix and the hottest source lines.  usage: ncu_summary.py REP"""
import csv
import io
import subprocess
import sys
from collections import Counter, defaultdict

rep = sys.argv[1]


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(ncu("--page", "details", "--csv"))))
want = {"Duration", "Compute (SM) Throughput", "Memory Throughput", "DRAM Throughput", "Issue Slots Busy",
        "Executed Ipc Active", "No Eligible", "Active Warps Per Scheduler", "Eligible Warps Per Scheduler",
        "Registers Per Thread", "Achieved Occupancy", "Waves Per SM", "L1/TEX Hit Rate", "L2 Hit Rate"}
iN, iU, iV = det[0].index("Metric Name"), det[0].index("Metric Unit"), det[0].index("Metric Value")
for r in det[1:]:
    if len(r) > iV and r[iN] in want:
        print(f"{r[iN]:32s} {r[iV]:>12s} {r[iU]}")
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): x for k, x in zip(h, v)
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
tot = sum(float(x) for x in st.values() if x.replace('.', '').isdigit())
print("stalls:", ", ".join(f"{k} {100*float(x)/tot:.0f}%" for k, x in sorted(st.items(), key=lambda kv: -float(kv[1]))[:8]))
for k, x in zip(h, v):
    if k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.sum",
             "smsp__sass_inst_executed_op_shared_ld.sum", "smsp__sass_inst_executed_op_local_ld.sum"):
        print(k, x)
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh = sass[1]
iI, iSrc = hh.index("Instructions Executed"), hh.index("Source")
c = Counter()
for r in sass[2:]:
    if len(r) > iI and r[iI].isdigit():
        t = r[iSrc].split()
        op = t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "")
        c[op.split(".")[0]] += int(r[iI])
print("mix:", ", ".join(f"{k} {n/1e6:.2f}M" for k, n in c.most_common(14)), f"| total {sum(c.values())/1e6:.2f}M")
cs = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
agg = defaultdict(lambda: [0, 0, ""])
cur = None
for r in cs:
    if len(r) >= 2 and r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    try:
        ln, s_, ins = int(r[0]), int(r[4]), int(r[7])
    except (ValueError, IndexError):
        continue
    a = agg[(cur, ln)]
    a[0] += s_
    a[1] += ins
    a[2] = r[1].strip()[:80]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{a[0]:5d} {a[1]:9d} {k[0]}:{k[1]} {a[2]}")
