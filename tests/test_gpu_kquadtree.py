"""Leaf-span tile kernels of the K quadtree (csrc/reduce.cu: hxf_span_mask / pack / unpack,
hxf_fixed_fold) against plain torch indexing, and distributed.reduce_scatter_quadtree on
one rank against the dense accumulator (second part)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _partition(units=9, leaf=6):
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs
    cfg = configs.cube_cluster(units, 13, "sp")
    return hx.build_partition(cfg.system, leaf_size=leaf), cfg.system.n_functions


def _random_fixed(n, seed, band):
    g = torch.Generator().manual_seed(seed)
    K = torch.randint(-2**45, 2**45, (n, n), generator=g, dtype=torch.int64)
    i = torch.arange(n)
    K[(i[:, None] - i[None, :]).abs() > band] = 0
    K[n - 3:, :2] = 5
    return K


@pytest.mark.parametrize("units,leaf", [(9, 6), (20, 10), (5, 3)])
def test_span_mask_pack_unpack_round_trip(units, leaf):
    from paper_1401_6961_b200 import distributed
    part, n = _partition(units, leaf)
    flo, fhi = distributed.leaf_function_ranges(part)
    nl = len(flo)
    Kh = _random_fixed(n, 5 + units, band=2 * leaf)
    K = Kh.cuda()
    flo_d, fhi_d = torch.from_numpy(flo).cuda(), torch.from_numpy(fhi).cuda()
    ops = distributed._NativeSpanOps
    m = ops.mask(K, flo_d, fhi_d).cpu().numpy().reshape(nl, nl)
    ref = np.zeros((nl, nl), dtype=np.uint8)
    for r in range(nl):
        for c in range(nl):
            ref[r, c] = int((Kh[flo[r]:fhi[r], flo[c]:fhi[c]] != 0).any())
    assert np.array_equal(m, ref)
    assert 0 < ref.sum() < nl * nl
    # pack every row span, then unpack a row range into a zeroed row block
    md = torch.from_numpy(ref.reshape(-1)).cuda()
    nf = (fhi - flo).astype(np.int64)
    sizes = (ref.astype(np.int64) * np.outer(nf, nf)).reshape(-1)
    off = np.concatenate([[0], np.cumsum(sizes)])
    off_d = torch.from_numpy(off).cuda()
    buf = torch.full((int(off[-1]),), -1, dtype=torch.int64, device="cuda")
    ops.move(K, 0, flo_d, fhi_d, 0, nl, md, off_d, 0, buf, True)
    bh = buf.cpu()
    for r in range(nl):
        for c in range(nl):
            if ref[r, c]:
                a = off[r * nl + c]
                assert torch.equal(bh[a:a + nf[r] * nf[c]].view(nf[r], nf[c]), Kh[flo[r]:fhi[r], flo[c]:fhi[c]])
    r0, r1 = nl // 3, nl - 1
    f0, f1 = int(flo[r0]), int(fhi[r1 - 1])
    rows = torch.zeros((f1 - f0, n), dtype=torch.int64, device="cuda")
    a0 = int(off[r0 * nl])
    ops.move(rows, f0, flo_d, fhi_d, r0, r1, md, off_d, a0, buf[a0:int(off[r1 * nl])].clone(), False)
    assert torch.equal(rows.cpu(), Kh[f0:f1])


def test_fixed_fold_is_exact():
    from paper_1401_6961_b200 import distributed
    Kh = _random_fixed(61, 3, band=61)
    K = Kh.cuda()
    distributed._NativeSpanOps.fold(K)
    assert torch.equal(K.cpu(), Kh + Kh.t())


@pytest.mark.parametrize("sym", [False, True])
def test_reduce_scatter_one_rank_matches_the_build(sym):
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs, distributed, exchange
    cfg = configs.cube_cluster(24, 5, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=cfg.leaf_size)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=cfg.tau_ovlp)
    P = torch.from_numpy(cfg.P).cuda()
    n = cfg.n_functions
    Pt = hx.build_matrix_tree(P, part)
    K1 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, True, None, K_out=K1)
    K = torch.empty((n, n), dtype=torch.float64, device="cuda")
    block, tree, c, stats = distributed.exchange_sharded_rows(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, K)
    assert (block.f0, block.f1) == (0, n)
    tol = 4e-16 * float(K1.abs().max()) if sym else 0.0
    assert float((block.dense() - K1).abs().max()) <= tol
    # the quadtree's leaf level is exactly the nonzero leaf tiles of K; the root is occupied
    flo, fhi = distributed.leaf_function_ranges(part)
    Kh = K1.cpu().numpy()
    nl = len(flo)
    for r in range(0, nl, 3):
        for cc in range(0, nl, 5):
            nz = bool((Kh[flo[r]:fhi[r], flo[cc]:fhi[cc]] != 0).any())
            assert bool(tree.leaf_mask[r, cc]) == nz or (tree.leaf_mask[r, cc] and not nz)
    assert tree.occupied(0, 0, 0) and tree.n_levels == len(part.levels)
    assert stats["bytes_packed"] == 8 * tree.stored_elements <= stats["bytes_dense"]
