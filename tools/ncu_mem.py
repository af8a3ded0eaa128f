"""Per-SASS-instruction memory traffic of one kernel in an .ncu-rep: global/shared
instructions with their L1 tag requests and L2 sectors, top N by tag requests.

usage: python tools/ncu_mem.py report.ncu-rep [top_n]
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--print-source", "sass", "--csv"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
rows = []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        tags = float(d["L1 Tag Requests Global"])
        sect = float(d["L2 Theoretical Sectors Global"])
        ins = float(d["Instructions Executed"])
    except ValueError:
        continue
    rows.append((d["Source"].strip(), ins, tags, sect, float(d["Warp Stall Sampling (All Samples)"])))
ti = sum(x[1] for x in rows)
tt = sum(x[2] for x in rows)
ts = sum(x[3] for x in rows)
print(f"warp instructions {ti:.4g}; L1 tag requests (global) {tt:.4g}; L2 theoretical sectors {ts:.4g}")
for src, ins, tags, sect, smp in sorted(rows, key=lambda x: -x[2])[:top]:
    if tags == 0:
        break
    print(f"{100 * tags / tt:5.1f}% tags  {tags / max(ins, 1):5.1f} tags/inst  {sect / max(ins, 1):5.1f} sect/inst  "
          f"{ins:10.4g} inst  {src[:70]}")
