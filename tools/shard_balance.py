"""Multi-GPU load balance measured on one GPU: the shards of an N-way plan run
one after another; each shard's device K-build time is what rank r would spend.

usage: python tools/shard_balance.py [config=c5] [worlds=2,4,8] [strategies=cyclic,contiguous]

Prints one JSON line per (world, strategy): per-shard ms and surviving quartets,
max/mean, and the predicted strong-scaling efficiency T_1 / (N * max_r T_r)
(the K all-reduce not included).  Sum of the shards' quartets must equal the
unsharded build's (checked).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1401_6961_b200 as hx  # noqa: E402
from paper_1401_6961_b200 import configs, distributed, exchange  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    worlds = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]
    strategies = (sys.argv[3] if len(sys.argv) > 3 else "balanced,hashed,cyclic,contiguous").split(",")
    cfg = configs.make(name, host_density=False) if name in ("c3", "c4", "c5") else configs.make(name)
    part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
    part.device(0)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
    n = cfg.n_functions
    P = configs.decay_density_device(cfg.system, cfg.density_seed) if cfg.P is None else \
        torch.as_tensor(cfg.P, device="cuda")
    Kb = torch.empty((n, n), dtype=torch.int64, device="cuda")

    def build(shard=None):
        Pt = hx.build_matrix_tree(P, part)
        _, c, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, True, None,
                                        K_out=Kb, shard=shard, symmetrize=False, K_fixed=True)
        torch.cuda.synchronize()
        t = exchange.last_timings()
        del Pt
        return t[4], int(c.eri_shell_quartets)

    build()
    t1, q1 = min(build() for _ in range(2))
    print(json.dumps({"config": name, "world": 1, "k_build_ms": t1, "quartets": q1}), flush=True)
    for world in worlds:
        for strategy in strategies:
            Pt = hx.build_matrix_tree(P, part)
            strat, _, rest = strategy.partition(":")
            mt, _, gp = rest.partition(":")
            tp = time.perf_counter()
            level, sel = distributed.plan(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, world,
                                          strategy=strat, min_tasks_per_rank=int(mt) if mt else None,
                                          K_scratch=Kb.view(torch.float64),
                                          groups_per_rank=int(gp) if gp else 16)
            plan_s = time.perf_counter() - tp
            del Pt
            ms, qs = [], []
            for b, e, s in sel:
                t, q = build((level, b, e, s))
                n_front = e
                ms.append(t)
                qs.append(q)
            assert sum(qs) == q1, (sum(qs), q1)
            print(json.dumps({"config": name, "world": world, "strategy": strategy, "cut_level": level, "frontier": n_front, "plan_s": plan_s,
                              "shard_ms": ms, "shard_quartets": qs,
                              "max_over_mean": max(ms) / (sum(ms) / len(ms)),
                              "predicted_efficiency": t1 / (world * max(ms))}), flush=True)


if __name__ == "__main__":
    main()
