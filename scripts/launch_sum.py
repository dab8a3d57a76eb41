"""Sum per-kernel durations of an ncu --metrics gpu__time_duration.sum --csv log."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = {}
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6}.get(d["Metric Unit"], 1.0)
        a = agg.setdefault(d["Kernel Name"][:70], [0.0, 0])
        a[0] += v
        a[1] += 1
for k, (v, n) in sorted(agg.items(), key=lambda x: -x[1][0])[:20]:
    print(f"{v / 1e3:10.3f} ms  n={n:5d}  {k}")
