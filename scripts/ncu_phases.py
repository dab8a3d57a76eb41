"""Executed warp instructions and stall samples per source line range (phases of
tile_compute) from an ncu report: python scripts/ncu_phases.py rep iters 'Y:480-505' ..."""
import csv
import io
import subprocess
import sys

rep, iters = sys.argv[1], int(sys.argv[2])
ranges = []
for a in sys.argv[3:]:
    name, r = a.split(":")
    lo, hi = r.split("-")
    ranges.append((name, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur = None
fname = None
agg = {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        continue
    if r[2].startswith("0x") and cur:
        try:
            e, smp = int(r[7] or 0), int(r[4] or 0)
        except ValueError:
            continue
        name = "other(" + cur[0] + ")"
        if cur[0] == "fused.cu":
            for n, lo, hi in ranges:
                if lo <= cur[1] <= hi:
                    name = n
                    break
        a = agg.setdefault(name, [0, 0])
        a[0] += e
        a[1] += smp
te = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
for k, (e, smp) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:32s} inst {100 * e / te:5.1f}% ({e / iters / 1e6:6.1f}M/iter)  samples {100 * smp / ts:5.1f}%")
