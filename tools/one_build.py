"""One exchange build of a BASELINE config (for ncu launch lists / captures).

usage: python tools/one_build.py c3 [naive|fourfold] [n_units] [repeats]
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_6961_b200 as hx  # noqa: E402
from paper_1401_6961_b200 import configs, exchange  # noqa: E402

name = sys.argv[1]
mode = sys.argv[2] if len(sys.argv) > 2 else "fourfold"
units = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3] != "-" else None
reps = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = configs.make(name, **({} if units is None else {"n_units": units}))
part = hx.build_partition(cfg.system, cfg.leaf_size)
pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
for _ in range(reps):
    Pt = hx.build_matrix_tree(cfg.P, part)
    K, c, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz",
                                    "eightfold" if mode == "eightfold" else mode == "fourfold")
    t = exchange.last_timings()
    print(name, mode, "quartets", c.eri_shell_quartets, "prim", c.prim_quartets,
          "stages_ms", [round(x, 2) for x in t], flush=True)
for k in range(16):
    if c.class_quartets[k] and os.environ.get("ONE_BUILD_CLASSES"):
        print(f"class {k:2d} ({k >> 3}{(k >> 2) & 1}{(k >> 1) & 1}{k & 1}) quartets {c.class_quartets[k]:.3e} "
              f"prim {c.class_prim_quartets[k]:.3e} prim/q {c.class_prim_quartets[k] / c.class_quartets[k]:.2f}")
