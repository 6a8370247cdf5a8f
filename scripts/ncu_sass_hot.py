"""Hottest SASS instructions of an ncu report with their dominant stall
reasons.  usage: ncu_sass_hot.py REP [N]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
iS, iA, iN = hdr.index("Source"), hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data = []
for idx, r in enumerate(rows[2:]):
    try:
        s = int(r[iN])
    except (ValueError, IndexError):
        continue
    data.append((s, idx, r))
tot = sum(d[0] for d in data)
print("total samples", tot)
for s, idx, r in sorted(data, key=lambda d: -d[0])[:n]:
    st = sorted(((int(r[i] or 0), hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
    print(f"{s:6d} #{idx:5d} {r[iS].strip()[:60]:60s} " + " ".join(f"{k}:{v}" for v, k in st if v))
