"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) per kernel name."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    v = float(d["Metric Value"].replace(",", ""))
    unit = d["Metric Unit"]
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
          "second": 1e3, "s": 1e3}.get(unit, 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v[1]:10.3f} ms {100 * v[1] / tot:5.1f}%  n={v[0]:5d}  {k[:110]}")
print(f"total {tot:.3f} ms")
