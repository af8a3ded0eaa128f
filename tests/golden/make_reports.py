"""Golden run reports from the REFERENCE's own harness (build container only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_reports.py

Writes tests/golden/reports.json: for each case, the reference report's
system block, counters, case occurrences, k_frobenius and comparison (timing and
timestamp fields dropped).  tests/test_harness.py checks the device harness
against it on the GPU.
"""
import json
import os

from hexfock.cli import RunConfig, run

CASES = [
    dict(system="water:3", mode="symmetry", reference="naive"),
    dict(system="water:2", mode="naive"),
    dict(system="water:2", mode="symmetry", tau_2e=1e-6, bound="literal"),
    dict(system="water:2", mode="naive", order="input", density="exp:gamma=1.0"),
    dict(system="water:1", mode="dense-screened", tau_ovlp=0.0),
]

out = []
for kw in CASES:
    r = run(RunConfig(**kw))
    for k in ("generated_at", "wall_seconds"):
        del r[k]
    out.append({"kwargs": kw, "report": r})
with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "reports.json"), "w") as fh:
    json.dump(out, fh, indent=1, sort_keys=True)
