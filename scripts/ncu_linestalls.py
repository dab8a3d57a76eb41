"""Per-source-line stall breakdown from an ncu report:
    python scripts/ncu_linestalls.py rep.ncu-rep [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 20
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
names = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
idx = {n: hdr.index(n) for n in names}
iS = hdr.index("Warp Stall Sampling (All Samples)")
cur, fname, agg, src = None, None, {}, {}
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) <= iS or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1].strip()[:70]
        continue
    if r[2].startswith("0x") and cur:
        a = agg.setdefault(cur, {n: 0 for n in names} | {"all": 0})
        for n, i in idx.items():
            try:
                a[n] += int(r[i] or 0)
            except ValueError:
                pass
        try:
            a["all"] += int(r[iS] or 0)
        except ValueError:
            pass
tot = sum(a["all"] for a in agg.values()) or 1
for k, a in sorted(agg.items(), key=lambda x: -x[1]["all"])[:top]:
    parts = sorted(((v, n[6:]) for n, v in a.items() if n != "all" and v), reverse=True)[:4]
    print(f"{k[0][:10]}:{k[1]:5d} {100 * a['all'] / tot:5.1f}% " + " ".join(f"{n}={100 * v / max(a['all'], 1):.0f}%"
                                                                           for v, n in parts) + f" | {src.get(k, '')}")
