"""Top SASS lines by warp-stall samples of an ncu report (source page, sass view).

    python tools/ncu_hot.py report.ncu-rep [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for i, r in enumerate(rows[2:]):
    try:
        data.append((float(r[wi]), i, r[si].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(x for x, _, _ in data) or 1.0
for x, i, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * x / tot:5.1f}%  [{i:4d}] {src}")
