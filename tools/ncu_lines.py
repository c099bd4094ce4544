"""Aggregate an ncu report's source page by CUDA source line.

python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] in ("", "Function Name"):
        continue
    rows.append((fname, r))
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


tot = sum(f(r[iS]) for _, r in rows) or 1
totE = sum(f(r[iE]) for _, r in rows) or 1
print(f"samples {tot:.0f} instructions {totE:.3g}")
for fn, r in sorted(rows, key=lambda x: -f(x[1][iS]))[:top]:
    print(f"{f(r[iS]) / tot * 100:5.1f}% {f(r[iE]) / totE * 100:5.1f}%  {fn}:{r[0]:>5} {r[1].strip()[:90]}")
