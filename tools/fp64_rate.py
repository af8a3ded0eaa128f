"""Per-kernel FP64 rate from an ncu --csv metric list (SURVEY.md 8(d) ncu recipe).

usage: python tools/fp64_rate.py launches.csv [peak_tflops] [classes.log]
FP64 flops = dadd + dmul + 2 dfma thread instructions; rate = flops / kernel time.
With the one_build.py class log, also executed FP64 flops per primitive quartet.
"""
import collections
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
peak = float(sys.argv[2]) if len(sys.argv) > 2 else 36.6
hdr = None
per = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    m, u = d["Metric Name"], d["Metric Unit"]
    v = float(d["Metric Value"].replace(",", ""))
    if m == "gpu__time_duration.sum":
        v *= {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "nsecond": 1e-9}[u]
        cnt[name] += 1
    if m.startswith("dram__bytes"):
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
    if "pct" in m:
        per[name][m + "_wsum"] += v * per[name]["_last_t"] if False else 0.0
    per[name][m] += v
prims = {}
if len(sys.argv) > 3:
    for line in open(sys.argv[3]):
        mm = re.match(r"class\s+(\d+) \((\d{4})\) quartets (\S+) prim (\S+)", line)
        if mm:
            prims["k_eri<%s, %s, %s, %s>" % tuple(mm.group(2))] = float(mm.group(4))
tot_f = tot_t = 0.0
print(f"{'kernel':24s} {'n':>4s} {'time ms':>9s} {'FP64 TF/s':>9s} {'% peak':>7s} {'DRAM GB/s':>9s} {'flop/prim':>9s}")
for name, d in sorted(per.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    t = d["gpu__time_duration.sum"]
    f = (d["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"] + d["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]
         + 2 * d["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"])
    b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    fp = f"{f / prims[name]:9.1f}" if name in prims else ""
    if name.startswith("k_eri"):
        tot_f += f
        tot_t += t
    print(f"{name[:24]:24s} {cnt[name]:4d} {1e3 * t:9.2f} {f / t / 1e12:9.2f} {100 * f / t / 1e12 / peak:7.1f} "
          f"{b / t / 1e9:9.1f} {fp}")
if tot_t:
    print(f"ERI stage (all k_eri): {tot_f / tot_t / 1e12:.2f} TFLOP/s executed FP64 = {100 * tot_f / tot_t / 1e12 / peak:.1f}% of {peak} TF/s")
