"""Per-source-line stall samples and executed instructions from an ncu report
(--import-source on):  python scripts/ncu_lines.py report.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
lines = []
cur = None
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        try:
            lines.append([fname, int(r[0]), r[1].strip()[:90], int(r[4] or 0), int(r[7] or 0)])
        except ValueError:
            pass
tot = sum(l[3] for l in lines) or 1
toti = sum(l[4] for l in lines) or 1
print(f"total samples {tot}, executed warp instructions {toti}")
for l in sorted(lines, key=lambda l: -l[3])[:top]:
    print(f"{l[0]}:{l[1]:5d} {100 * l[3] / tot:5.1f}% samp {100 * l[4] / toti:5.1f}% inst | {l[2]}")
