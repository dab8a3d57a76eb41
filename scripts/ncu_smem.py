"""Shared-memory wavefronts (actual / ideal) per source line from an ncu report."""
import csv
import io
import subprocess
import sys

rep, iters = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 10
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
iW, iI = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
cur, fname, agg, src = None, None, {}, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= iI or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:80]
        continue
    if r[2].startswith("0x") and cur:
        try:
            w, wi = int(r[iW] or 0), int(r[iI] or 0)
        except ValueError:
            continue
        a = agg.setdefault(cur, [0, 0])
        a[0] += w
        a[1] += wi
tw = sum(v[0] for v in agg.values())
ti = sum(v[1] for v in agg.values())
print(f"shared wavefronts/iter {tw / iters / 1e6:.1f}M (ideal {ti / iters / 1e6:.1f}M)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:25]:
    print(f"{k[0][:10]}:{k[1]:5d} {v[0] / iters / 1e6:6.2f}M ideal {v[1] / iters / 1e6:6.2f}M | {src.get(k, '')}")
