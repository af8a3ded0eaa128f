"""Host vs device Hilbert reordering on BASELINE config 5's system.

python tools/prep_timing.py [out.json]: generates a 4096-molecule water-like
cluster (16384 shells), times inputs.hilbert_order (host pre-pass, reference
basis.py:309-331) once and prep.hilbert_keys_and_perm (device, host buffers in
and out) over 20 calls after warm-up, checks the permutations are equal; then the
same for the partition build (quadtree.py:90-113; device time includes the Span
tree the wrapper rebuilds on the host)."""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1401_6961_b200 import basis, inputs, prep, quadtree  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    s = inputs.generate_cluster(4096, seed=5)
    c = np.array([sh.center for sh in s.shells])
    t0 = time.perf_counter()
    _, p_h = inputs.hilbert_order(s)
    host_s = time.perf_counter() - t0
    for _ in range(3):
        prep.hilbert_keys_and_perm(c, 10)
    t0 = time.perf_counter()
    reps = 20
    for _ in range(reps):
        _, p_d = prep.hilbert_keys_and_perm(c, 10)
    dev_s = (time.perf_counter() - t0) / reps
    rec = {"shells": len(s.shells), "bits": 10, "host_hilbert_order_s": host_s,
           "device_hilbert_order_s": dev_s, "speedup": host_s / dev_s,
           "perm_equal": bool(np.array_equal(p_h, p_d)),
           "note": "device time includes the H2D of the centres and D2H of the permutation"}
    s2, _ = inputs.hilbert_order(s)
    t0 = time.perf_counter()
    ph = quadtree.build_partition(s2, 10)
    rec["host_build_partition_s"] = time.perf_counter() - t0
    prep.build_partition_device(s2, 10)
    t0 = time.perf_counter()
    for _ in range(reps):
        pd = prep.build_partition_device(s2, 10)
    rec["device_build_partition_s"] = (time.perf_counter() - t0) / reps
    rec["partition_levels_equal"] = [[(x.shell_lo, x.shell_hi) for x in lv] for lv in ph.levels] == \
        [[(x.shell_lo, x.shell_hi) for x in lv] for lv in pd.levels]
    print(json.dumps(rec))
    if out:
        with open(out, "w") as f:
            json.dump(rec, f, indent=1)


if __name__ == "__main__":
    main()
