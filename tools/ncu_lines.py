"""Per-CUDA-source-line warp-stall samples of an ncu report (mixed
cuda,sass source page).  Usage: python tools/ncu_lines.py rep [n]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
f = None
agg = {}
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if not r or r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "":
        try:
            s = float(r[4])
        except ValueError:
            s = 0.0
        if s > 0:
            agg[(f, r[0], r[1][:100])] = agg.get((f, r[0], r[1][:100]), 0) + s
tot = sum(agg.values())
print("samples", tot)
for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:n]:
    print(f"{v:7.0f} {v / tot * 100:5.1f}% {k[0]}:{k[1]} {k[2]}")
