"""Tile sparsity of a full exchange K and the cost of the block-sparse reduction
passes: python tools/k_sparsity.py c5 [bs ...] [--out f.json].

One fourfold build into the int64 fixed-point accumulator, then per tile size the
fraction of nonzero tiles (= the all-reduce bytes the sparse path moves vs dense)
and the device time of mask + slots + pack + unpack (CUDA events, after a warm-up)."""

import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1401_6961_b200 as hx  # noqa: E402
from paper_1401_6961_b200 import configs, distributed, exchange  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
out = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
if out in args:
    args.remove(out)
name = args[0] if args else "c5"
sizes = [int(a) for a in args[1:]] or [32, 64, 128]
cfg = configs.make(name)
part = hx.build_partition(cfg.system, cfg.leaf_size)
pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
Pt = hx.build_matrix_tree(cfg.P, part)
n = cfg.P.shape[0]
Kfx = torch.zeros(n, n, dtype=torch.int64, device="cuda")
exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, True, None, K_out=Kfx,
                      symmetrize=False, K_fixed=True)
torch.cuda.synchronize()
OPS = distributed._NativeBlockOps
rows = []
for bs in sizes:
    times = []
    for rep in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        m = OPS.mask(Kfx, bs)
        slot, nblk = OPS.slots(m)
        buf = OPS.pack(Kfx, bs, m, slot, nblk)
        K2 = Kfx.clone() if rep == 0 else None
        b.record()
        torch.cuda.synchronize()
        times.append(a.elapsed_time(b))
        if rep == 0:
            K2.zero_()
            OPS.unpack(K2, bs, m, slot, buf)
            assert torch.equal(K2, Kfx)
            del K2
        del buf
    rows.append({"bs": bs, "tiles": int(m.numel()), "tiles_nonzero": nblk,
                 "fraction": nblk / m.numel(), "bytes_sparse": nblk * bs * bs * 8 + int(m.numel()),
                 "bytes_dense": n * n * 8, "mask_slots_pack_ms": min(times[1:])})
rec = {"config": name, "functions": n, "rows": rows}
print(json.dumps(rec))
if out:
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
