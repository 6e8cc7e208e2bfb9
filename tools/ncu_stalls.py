"""Aggregate the per-instruction warp-stall samples of an ncu capture (source page, SASS):
total by stall reason and the hottest instructions.  python tools/ncu_stalls.py rep [n]"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[1], rows[2:]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: sum(float(x[hdr.index(r)] or 0) for x in data) for r in reasons}
allS = sum(tot.values())
print("stall samples by reason:")
for r, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]:
    print(f"  {r:24s} {100 * v / allS:5.1f}%")
iS = hdr.index("Warp Stall Sampling (All Samples)")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
print("hottest instructions:")
for i in sorted(sorted(range(len(data)), key=lambda i: -float(data[i][iS] or 0))[:n]):
    x = data[i]
    top = max(reasons, key=lambda r: float(x[hdr.index(r)] or 0))
    print(f"  {i:5d} {100 * float(x[iS]) / allS:5.1f}% {top:20s} {x[1].strip()[:70]}")
