"""Per-source-line instruction and stall-sample totals of one kernel in an .ncu-rep.

usage: python tools/ncu_lines.py report.ncu-rep [top_n]
(the report must be captured with --import-source on from a -lineinfo build)
"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--print-source", "cuda,sass", "--csv"],
                     capture_output=True, text=True).stdout
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = []
fname = None
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        ins = float(r[hdr.index("Instructions Executed")])
        smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except (ValueError, IndexError):
        continue
    rows.append((fname, int(r[0]), r[1][:90], ins, smp))
ti = sum(x[3] for x in rows) or 1
ts = sum(x[4] for x in rows) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts:.4g}")
for f, ln, src, ins, smp in sorted(rows, key=lambda x: -x[3])[:top]:
    print(f"{100 * ins / ti:5.1f}% ins {100 * smp / ts:5.1f}% smp  {f}:{ln}  {src}")
