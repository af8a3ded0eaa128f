"""Per-build DRAM traffic of the path's kernel families from an ncu metric list.

usage: python tools/ncu_dram.py launches.csv workload mode builds > profiles/rNN_ncu_<workload>_dram.json

The csv comes from
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:"k_eri|k_screen2|k_expand|k_bin|DeviceRadixSort" --csv --log-file launches.csv \
      python tools/one_build.py <workload> <mode> - <builds>
bench.py quotes k_eri's bytes per build as roofline.traffic (ncu replays are
cold-cache and serialised: bytes are meaningful, times only as shares).
"""
import json
import sys

sys.path.insert(0, __file__.rsplit("/", 2)[0])
from tools.tau_sweep import _UNIT  # noqa: E402
import csv  # noqa: E402

path, workload, mode, builds = sys.argv[1], sys.argv[2], sys.argv[3], int(sys.argv[4])
# k_binb_classify / k_binb_scatter: survivor binning; DeviceRadixSort: the leaf-task order (cub, keys only)
fam = {"k_eri": {}, "k_screen2": {}, "k_expand": {}, "k_binb_classify": {}, "k_binb_scatter": {}, "DeviceRadixSort": {}}
hdr = None
launches = {k: set() for k in fam}
for r in csv.reader(open(path)):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    f = next((k for k in fam if k in d["Kernel Name"]), None)
    if f is None:
        continue
    launches[f].add(d["ID"])
    v = float(d["Metric Value"].replace(",", "")) * _UNIT.get(d["Metric Unit"], 1.0)
    fam[f][d["Metric Name"]] = fam[f].get(d["Metric Name"], 0.0) + v
out = {"workload": workload, "mode": mode, "builds_captured": builds, "source": path.rsplit("/", 1)[-1]}
for k, m in fam.items():
    b = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    t = m.get("gpu__time_duration.sum", 0.0)
    out[k] = {"launches_per_build": len(launches[k]) / builds, "dram_bytes_per_build": b / builds,
              "dram_read_bytes_per_build": m.get("dram__bytes_read.sum", 0.0) / builds,
              "ncu_ms_per_build": 1e3 * t / builds, "ncu_dram_gbs": b / t / 1e9 if t else None}
print(json.dumps(out, indent=1))
