"""Top SASS instructions by warp-stall samples of an ncu report, with the
CUDA source line each maps to.  Usage: python tools/ncu_stalls.py rep [n]"""
import csv
import subprocess
import sys

def fl(s):
    try:
        return float(s)
    except ValueError:
        return 0.0


rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if "Address" in r and "Source" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
tot = sum(fl(r[iS]) for r in data)
print("samples", tot, "instructions", len(data))
for r in sorted(data, key=lambda r: -fl(r[iS]))[:n]:
    print(f"{fl(r[iS]):6.0f} {fl(r[iS]) / tot * 100:5.1f}% ex={r[iE]:>6} {r[1][:100]}")
