"""Block-sparse reduction tile kernels (csrc/reduce.cu) on the
GPU: tile masks against torch, pack/unpack round trips, and a two-shard reduction
done on one device (pack both shards' real exchange accumulators, add the buffers
as the all-reduce would, unpack) equal to the dense sum bit for bit."""

import numpy as np
import pytest
import torch

from paper_1401_6961_b200 import configs, distributed, exchange
import paper_1401_6961_b200 as hx

pytestmark = pytest.mark.gpu
OPS = distributed._NativeBlockOps


def _torch_mask(K, bs):
    n = K.shape[0]
    nb = (n + bs - 1) // bs
    pad = torch.zeros(nb * bs, nb * bs, dtype=K.dtype, device=K.device)
    pad[:n, :n] = K
    return (pad.view(nb, bs, nb, bs) != 0).any(dim=3).any(dim=1).reshape(-1).to(torch.uint8)


def _sparse(n, seed, band=60):
    g = torch.Generator().manual_seed(seed)
    K = torch.randint(-2**50, 2**50, (n, n), generator=g, dtype=torch.int64)
    i = torch.arange(n)
    K[(i[:, None] - i[None, :]).abs() > band] = 0
    K[n - 1, 0] = 1                                   # a lone corner entry
    return K.cuda()


@pytest.mark.parametrize("n,bs", [(1, 1), (7, 64), (300, 1), (1000, 7), (1000, 64), (1031, 128)])
def test_mask_and_roundtrip(n, bs):
    K = _sparse(n, n + bs)
    m = OPS.mask(K, bs)
    assert torch.equal(m, _torch_mask(K, bs))
    slot, nblk = OPS.slots(m)
    assert nblk == int(m.sum()) and int(slot[-1]) == nblk
    buf = OPS.pack(K, bs, m, slot, nblk)
    K2 = torch.zeros_like(K)
    OPS.unpack(K2, bs, m, slot, buf)
    assert torch.equal(K2, K)


def test_two_shard_reduction_of_real_exchange():
    cfg = configs.make("c3")
    part = hx.build_partition(cfg.system, cfg.leaf_size)
    pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    Pt = hx.build_matrix_tree(cfg.P, part)
    n = cfg.P.shape[0]
    shards = distributed.plan(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, 2)
    level, ranges = shards
    parts, scale = [], None
    for r in range(2):
        b, e, stride = ranges[r]
        Kfx = torch.zeros(n, n, dtype=torch.int64, device="cuda")
        (_, S), _, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, True, None,
                                             K_out=Kfx, shard=(level, b, e, stride), symmetrize=False,
                                             K_fixed=True)
        assert scale in (None, S)
        scale = S
        parts.append(Kfx)
    bs = 64
    m = torch.maximum(OPS.mask(parts[0], bs), OPS.mask(parts[1], bs))   # the uint8 MAX all-reduce
    slot, nblk = OPS.slots(m)
    buf = OPS.pack(parts[0], bs, m, slot, nblk) + OPS.pack(parts[1], bs, m, slot, nblk)  # the SUM
    K = parts[0].clone()
    OPS.unpack(K, bs, m, slot, buf)
    assert torch.equal(K, parts[0] + parts[1])
    print(f"c3 K tiles {bs}x{bs}: {nblk}/{m.numel()} nonzero")
