"""Host-side breakdown of one bench step (density tree, exchange, teardown).

usage: python tools/step_breakdown.py [c5] [fourfold|naive] [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1401_6961_b200 as hx  # noqa: E402
from paper_1401_6961_b200 import configs, exchange  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
sym = (sys.argv[2] if len(sys.argv) > 2 else "fourfold") == "fourfold"
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
cfg = configs.make(name, host_density=False) if name in ("c3", "c4", "c5") else configs.make(name)
dev = torch.device("cuda", 0)
P = cfg.P if cfg.P is not None else configs.decay_density_device(cfg.system, cfg.density_seed, dev)
if not torch.is_tensor(P):
    P = torch.from_numpy(P).to(dev)
part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
part.device(0)
pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
K = torch.empty_like(P)
torch.cuda.synchronize()
for r in range(reps):
    t0 = time.perf_counter()
    Pt = hx.build_matrix_tree(P, part)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    _, c, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, True, None, K_out=K)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    del Pt
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    st = exchange.last_timings()
    print(f"rep {r}: density {1e3*(t1-t0):.1f} ms  exchange {1e3*(t2-t1):.1f} ms (device total {st[4]:.1f}: "
          f"trav {st[0]:.1f} screen {st[1]:.1f} eri {st[2]:.1f} [kernels {st[5]:.1f} sort {st[6]:.1f}] epi {st[3]:.1f})  "
          f"teardown {1e3*(t3-t2):.1f} ms",
          flush=True)
