import sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_1401_6961_b200 as hx
from paper_1401_6961_b200 import configs, exchange
name = sys.argv[1]; units = int(sys.argv[2]) if len(sys.argv) > 2 else None
t = time.time()
cfg = configs.make(name, **({} if units is None else {"n_units": units}))
print("gen", name, cfg.n_shells, cfg.n_functions, f"{time.time()-t:.1f}s", flush=True)
t = time.time(); part = hx.build_partition(cfg.system, 10); print("part", len(part.levels), f"{time.time()-t:.2f}s", flush=True)
t = time.time(); pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp); print("pairtree", f"{time.time()-t:.2f}s", flush=True)
t = time.time(); Pt = hx.build_matrix_tree(cfg.P, part); print("ptree", f"{time.time()-t:.2f}s", flush=True)
for sym in (False, True):
    for rep in range(2):
        t = time.time()
        if sym: K, c = hx.build_exchange_symmetric(pairs, Pt, cfg.tau_2e)
        else: K, c = hx.build_exchange_naive(pairs, pairs, Pt, cfg.tau_2e)
        dt = time.time() - t
        tm = exchange.last_timings()
        print("sym" if sym else "naive", f"wall {dt*1e3:.1f} ms", "stages", [round(x,1) for x in tm], "quartets %.3e" % c.eri_shell_quartets, "primq %.3e" % c.prim_quartets, "rate %.3e q/s" % (c.eri_shell_quartets/(tm[4]/1e3)), "leaf", c.leaf_contractions, "visited", c.tasks_visited, "ties", c.ties_task, c.ties_leaf, flush=True)
