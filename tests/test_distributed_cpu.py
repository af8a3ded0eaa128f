"""Multi-rank host logic on CPU (gloo, world_size 2).

The device path shards the product-tree frontier at a cut level into
cyclic selections (distributed.split_cyclic: every world-th task from the
rank's index) or contiguous ranges (distributed.split_by_cost), each rank runs
its subtrees into a private K, work above the cut is counted by shard 0
only, and K / counters are summed by one all-reduce
(distributed.allreduce_partials).  Here the per-rank compute is the CPU
oracle (the checker) driven over the same frontier order the device uses
(parents in order, children in (a, cc, d, bb) order), so the sharding
semantics and the reduction plumbing are verified without a GPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hexfock_oracle as ho
from paper_1401_6961_b200 import configs, distributed


def test_split_by_cost_contiguous_balanced():
    costs = np.array([5, 1, 1, 1, 1, 1, 5, 1, 1, 3], dtype=float)
    for world in (1, 2, 3, 4, 7, 16):
        r = distributed.split_by_cost(costs, world)
        assert len(r) == world
        assert r[0][0] == 0 and r[-1][1] == len(costs)
        for (b0, e0), (b1, e1) in zip(r, r[1:]):
            assert e0 == b1 and b0 <= e0
    r = distributed.split_by_cost(np.ones(100), 4)
    assert [e - b for b, e in r] == [25, 25, 25, 25]
    assert distributed.split_by_cost(np.ones(0), 3) == [(0, 0), (0, 0), (0, 0)]


def test_split_cyclic_partitions_frontier():
    for n in (0, 1, 5, 64, 1000):
        for world in (1, 2, 3, 8):
            sel = distributed.split_cyclic(n, world)
            assert len(sel) == world
            got = sorted(i for b, e, s in sel for i in range(b, e, s))
            assert got == list(range(n))


def test_split_lpt_balances_group_costs():
    rng = np.random.default_rng(5)
    for world, groups in ((2, 32), (4, 64), (8, 128)):
        costs = rng.pareto(2.0, size=groups) + 0.1
        n = 20000
        sel = distributed.split_lpt(n, world, groups, costs)
        owners = np.stack([m for _, _, m in sel])
        assert np.array_equal(owners.sum(axis=0), np.ones(n))
        assert [b == 0 for b, _, _ in sel] == [True] + [False] * (world - 1)
        # every task of a group lands on one rank; rank loads within the LPT bound
        grp = distributed._owner(n, groups)
        load = np.zeros(world)
        for g in range(groups):
            ranks = {int(np.argmax(owners[:, t])) for t in np.nonzero(grp == g)[0]}
            assert len(ranks) <= 1
            if ranks:
                load[ranks.pop()] += costs[g]
        assert load.max() <= costs.sum() / world + costs.max() + 1e-12
    assert distributed.split_lpt(0, 3, 8, np.ones(8))[0][2].shape == (0,)


def test_split_hashed_partitions_frontier():
    for n in (0, 1, 5, 64, 5000):
        for world in (1, 2, 3, 8):
            sel = distributed.split_hashed(n, world)
            assert len(sel) == world
            assert [b == 0 for b, _, _ in sel] == [True] + [False] * (world - 1)  # top owner
            owners = np.stack([m for _, _, m in sel]) if n else np.zeros((world, 0))
            assert all(e == n for _, e, _ in sel)
            assert np.array_equal(owners.sum(axis=0), np.ones(n))
            if n >= 5000:
                assert owners.sum(axis=1).max() <= 1.1 * n / world


def test_counters_vector_roundtrip():
    class C:  # mimics the ctypes counters struct
        pass
    c = C()
    for i, k in enumerate(("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
                           "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
                           "tasks_expanded", "children_spawned", "links_culled_screening",
                           "links_culled_absent", "ties_task", "ties_leaf", "prim_quartets")):
        setattr(c, k, 10 * i + 1)
    c.case_tasks = list(range(9))
    c.case_leaf_tasks = list(range(9, 18))
    c.class_quartets = [0] * 16
    c.class_prim_quartets = [0] * 16
    c.culled_bound_ledger = 0.125
    out = distributed.counters_from_vector(distributed.counters_vector(c), True)
    assert out.tasks_visited == 1 and out.children_spawned == 71
    assert out.case_tasks["SPARSE"] == 8 and out.case_leaf_tasks["A"] == 9
    assert out.culled_bound_ledger == 0.125


# ------------------------------------------------------------ sharded oracle

def _frontier(st, tau, level, run):
    """Naive BFS to `level` in device order; visits above the cut go to `run`."""
    fr = [(st.pairs, st.Ptree, st.pairs)]
    # the root visit
    run.c.tasks_visited += 1
    b, p, k = fr[0]
    if _cull(run, b, p, k):
        return []
    if b.is_leaf and k.is_leaf:
        run.c.leaf_contractions += 1
        run.contract(b, p, k)
        return []
    run.c.tasks_expanded += 1
    for _ in range(level):
        nxt = []
        for b, p, k in fr:
            for a in range(len(b.row.kids())):
                for cc in range(len(b.col.kids())):
                    bch = b.child(a, cc)
                    for d in range(len(k.row.kids())):
                        pch = p.child(cc, d)
                        for bb in range(len(k.col.kids())):
                            kch = k.child(d, bb)
                            run.c.children_spawned += 1
                            run.c.tasks_visited += 1
                            if _cull(run, bch, pch, kch):
                                continue
                            if bch.is_leaf and kch.is_leaf:
                                run.c.leaf_contractions += 1
                                run.contract(bch, pch, kch)
                                continue
                            run.c.tasks_expanded += 1
                            nxt.append((bch, pch, kch))
        fr = nxt
    return fr


def _cull(run, b, p, k):
    c = run.c
    if b is None or p is None or k is None or b.pruned or k.pruned:
        c.tasks_culled_absent += 1
        return True
    import math
    if ho.sorted_product(math.sqrt(b.diag_norm), p.norm, math.sqrt(k.diag_norm)) <= run.tau:
        c.tasks_culled_screening += 1
        c.culled_bound_ledger += ho.culled_task_bound(b, p.norm, k)
        return True
    return False


def _expand_children(run, b, p, k):
    for a in range(len(b.row.kids())):
        for cc in range(len(b.col.kids())):
            bch = b.child(a, cc)
            for d in range(len(k.row.kids())):
                pch = p.child(cc, d)
                for bb in range(len(k.col.kids())):
                    run.c.children_spawned += 1
                    run.visit(bch, pch, k.child(d, bb))


def _sharded_run(st, tau, level, world, rank, strategy):
    top = ho._Naive(st.shells, st.P, st.P.shape[0], tau, "schwarz", True, False)
    frontier = _frontier(st, tau, level, top)
    if strategy == "hashed":
        _, _, m = distributed.split_hashed(len(frontier), world)[rank]
        picked = [t for t, keep in zip(frontier, m) if keep]
    elif strategy == "balanced":
        # distributed.plan(strategy="balanced") on the CPU: hashed task groups costed by
        # counters-only runs (every rank costs every world-th group, one all-reduce),
        # then longest-first onto ranks (group_costs + split_lpt)
        groups = 4 * world
        owner = distributed._owner(len(frontier), groups)
        cost = np.zeros(groups)
        for g in range(rank, groups, world):
            probe = ho._Naive(st.shells, st.P, st.P.shape[0], tau, "schwarz", False, False)
            for (b, p, k), o in zip(frontier, owner):
                if o == g:
                    _expand_children(probe, b, p, k)
            cost[g] = (distributed.COST_PER_QUARTET * probe.c.eri_shell_quartets
                       + distributed.COST_PER_LEAF_TASK * probe.c.leaf_contractions
                       + distributed.COST_PER_VISIT * probe.c.tasks_visited)
        t = torch.from_numpy(cost)
        if dist.is_initialized():
            dist.all_reduce(t)
        _, _, m = distributed.split_lpt(len(frontier), world, groups, t.numpy())[rank]
        picked = [t_ for t_, keep in zip(frontier, m) if keep]
    elif strategy == "cyclic":
        b0, e0, s0 = distributed.split_cyclic(len(frontier), world)[rank]
        picked = frontier[b0:e0:s0]
    else:
        b0, e0 = distributed.split_by_cost(np.ones(len(frontier)), world)[rank]
        picked = frontier[b0:e0]
    mine = ho._Naive(st.shells, st.P, st.P.shape[0], tau, "schwarz", True, False)
    for b, p, k in picked:
        _expand_children(mine, b, p, k)
    if rank == 0:
        mine.K += top.K
        mine.c.merge(top.c)
    return mine


def _vec(c):
    return np.array([c.tasks_visited, c.tasks_culled_screening, c.tasks_culled_absent,
                     c.leaf_contractions, c.eri_shell_quartets, c.quartets_culled_leaf,
                     c.tasks_expanded, c.children_spawned, c.culled_bound_ledger], dtype=np.float64)


def _worker(rank, world, port, result_path, strategy):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = configs.cube_cluster(4, 7, "tiny")
    st = ho.Setup(cfg.system, cfg.P, tau_ovlp=1e-11, leaf_size=4)
    run = _sharded_run(st, 1e-8, 2, world, rank, strategy)
    K = torch.from_numpy(run.K.copy())
    vec = torch.from_numpy(_vec(run.c))
    distributed.allreduce_partials(K, vec)
    if rank == 0:
        np.savez(result_path, K=K.numpy(), vec=vec.numpy())
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,strategy", [(2, "hashed"), (2, "balanced"), (2, "cyclic"), (2, "contiguous")])
def test_gloo_sharded_build_equals_single_process(tmp_path, world, strategy):
    path = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(world, _free_port(), path, strategy), nprocs=world, join=True)
    res = np.load(path)
    cfg = configs.cube_cluster(4, 7, "tiny")
    st = ho.Setup(cfg.system, cfg.P, tau_ovlp=1e-11, leaf_size=4)
    K, c = st.naive(1e-8)
    assert np.abs(res["K"] - K).max() <= 1e-13
    ref = _vec(c)
    assert np.array_equal(res["vec"][:8], ref[:8])        # integer counters exact
    assert res["vec"][8] == pytest.approx(ref[8], rel=1e-12)


# ------------------------------------------------ block-sparse reduction (§8(f) f4)

class _TorchBlockOps:
    """CPU stand-in for the libhxf tile kernels (test checker only): the host
    logic of distributed.allreduce_fixed_sparse runs over gloo with these."""

    @staticmethod
    def _tiles(K, bs):
        n = K.shape[0]
        nb = (n + bs - 1) // bs
        pad = torch.zeros(nb * bs, nb * bs, dtype=K.dtype)
        pad[:n, :n] = K
        return pad.view(nb, bs, nb, bs).permute(0, 2, 1, 3).reshape(nb * nb, bs * bs)

    @classmethod
    def mask(cls, K, bs):
        return (cls._tiles(K, bs) != 0).any(dim=1).to(torch.uint8)

    @staticmethod
    def slots(m):
        slot = torch.zeros(m.numel() + 1, dtype=torch.int64)
        slot[1:] = torch.cumsum(m.to(torch.int64), 0)
        return slot, int(slot[-1])

    @classmethod
    def pack(cls, K, bs, m, slot, nblk):
        return cls._tiles(K, bs)[m.bool()].reshape(-1).clone()

    @classmethod
    def unpack(cls, K, bs, m, slot, buf):
        n = K.shape[0]
        nb = (n + bs - 1) // bs
        t = cls._tiles(K, bs)
        t[m.bool()] = buf.view(-1, bs * bs)
        full = t.view(nb, nb, bs, bs).permute(0, 2, 1, 3).reshape(nb * bs, nb * bs)
        K.copy_(full[:n, :n])


def _sparse_worker(rank, world, port, result_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    K = _rank_partial(rank)
    vec = torch.tensor([float(rank + 1)], dtype=torch.float64)
    K, vec, stats = distributed.allreduce_fixed_sparse(K, vec, block=8, ops=_TorchBlockOps)
    if rank == 0:
        np.savez(result_path, K=K.numpy(), vec=vec.numpy(), nz=stats["tiles_nonzero"], tiles=stats["tiles"])
    dist.barrier()
    dist.destroy_process_group()


def _rank_partial(rank, n=45):
    """Banded int64 partial with rank-specific tiles (some tiles nonzero on one rank only,
    entries cancelling to zero across ranks in one tile)."""
    g = torch.Generator().manual_seed(100 + rank)
    K = torch.randint(-2**40, 2**40, (n, n), generator=g, dtype=torch.int64)
    i = torch.arange(n)
    K[(i[:, None] - i[None, :]).abs() > 10] = 0
    if rank == 0:
        K[40:45, 0:3] = 7
        K[16:24, 24:32] = 5
    else:
        K[0:3, 40:45] = -3
        K[16:24, 24:32] = -5
    return K


def test_gloo_block_sparse_allreduce_equals_dense(tmp_path):
    path = str(tmp_path / "sparse.npz")
    mp.spawn(_sparse_worker, args=(2, _free_port(), path), nprocs=2, join=True)
    res = np.load(path)
    dense = (_rank_partial(0) + _rank_partial(1)).numpy()
    assert np.array_equal(res["K"], dense)
    assert res["vec"][0] == 3.0
    assert 0 < int(res["nz"]) < int(res["tiles"])        # the band leaves tiles out


# ------------------------------- K quadtree + row-owning reduce-scatter (§8(f) f4, second part)

class _TorchSpanOps:
    """CPU stand-in for the libhxf leaf-span tile kernels (test checker only): the host
    logic of distributed.reduce_scatter_quadtree runs over gloo with these."""

    @staticmethod
    def mask(K, flo, fhi):
        nl = flo.numel()
        m = torch.zeros(nl, nl, dtype=torch.uint8)
        for r in range(nl):
            for c in range(nl):
                m[r, c] = int((K[flo[r]:fhi[r], flo[c]:fhi[c]] != 0).any())
        return m.reshape(-1)

    @staticmethod
    def move(K, row_base, flo, fhi, r0, r1, m, off, off_base, buf, pack):
        nl = flo.numel()
        for r in range(r0, r1):
            for c in range(nl):
                if not m[r * nl + c]:
                    continue
                h, w = int(fhi[r] - flo[r]), int(fhi[c] - flo[c])
                a = int(off[r * nl + c]) - off_base
                tile = K[int(flo[r]) - row_base:int(fhi[r]) - row_base, int(flo[c]):int(fhi[c])]
                if pack:
                    buf[a:a + h * w] = tile.reshape(-1)
                else:
                    tile.copy_(buf[a:a + h * w].view(h, w))

    @staticmethod
    def fold(K):
        K.add_(K.t().clone())


def _span_partition():
    """A ragged partition: s and p shells mixed, leaf spans of 3..6 functions."""
    cfg = configs.cube_cluster(6, 11, "sp")
    import paper_1401_6961_b200 as hx
    return hx.build_partition(cfg.system, leaf_size=6), cfg.system.n_functions


def _span_partial(rank, n):
    g = torch.Generator().manual_seed(300 + rank)
    K = torch.randint(-2**40, 2**40, (n, n), generator=g, dtype=torch.int64)
    i = torch.arange(n)
    K[(i[:, None] - i[None, :]).abs() > 9] = 0
    K[n - 4:, :3] = 11 * (rank + 1)          # a far corner tile, one-sided
    if rank == 1:
        K[:5, :] = 0                         # rank 1 holds nothing in the first rows
    return K


def _scatter_worker(rank, world, port, result_path, fold):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    part, n = _span_partition()
    K = _span_partial(rank, n)
    block, tree, stats = distributed.reduce_scatter_quadtree(K, part, scale=20, fold=fold, ops=_TorchSpanOps)
    np.savez(result_path + f".{rank}.npz", rows=block.dense_fixed().numpy(), f0=block.f0, f1=block.f1,
             dense=block.dense().numpy(), leaf=tree.leaf_mask, top=tree.levels[0], l1=tree.levels[1],
             packed=stats["packed_elements"], owned=stats["bytes_owned"], nnz=tree.nnz_tiles,
             stored=tree.stored_elements)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("fold", [False, True])
def test_gloo_quadtree_reduce_scatter_rows(tmp_path, fold):
    path = str(tmp_path / "rs")
    mp.spawn(_scatter_worker, args=(2, _free_port(), path, fold), nprocs=2, join=True)
    part, n = _span_partition()
    parts = [_span_partial(r, n) for r in range(2)]
    if fold:
        parts = [p + p.t() for p in parts]
    full = (parts[0] + parts[1]).numpy()
    got = [np.load(path + f".{r}.npz") for r in range(2)]
    # the two ranks own disjoint, contiguous row ranges that cover every row
    assert int(got[0]["f0"]) == 0 and int(got[0]["f1"]) == int(got[1]["f0"]) and int(got[1]["f1"]) == n
    assert 0 < int(got[0]["f1"]) < n
    for g in got:
        f0, f1 = int(g["f0"]), int(g["f1"])
        assert np.array_equal(g["rows"], full[f0:f1])             # exact integer sum of the owner's rows
        scale = 2.0 ** -(20 + (1 if fold else 0))
        assert np.array_equal(g["dense"], full[f0:f1].astype(np.float64) * scale)
    # the quadtree: leaf occupancy = union of the ranks' nonzero leaf tiles, OR-ed upward
    flo, fhi = distributed.leaf_function_ranges(part)
    nl = len(flo)
    union = np.zeros((nl, nl), dtype=np.uint8)
    for p in parts:
        for r in range(nl):
            for c in range(nl):
                union[r, c] |= int((p[flo[r]:fhi[r], flo[c]:fhi[c]] != 0).any())
    assert np.array_equal(got[0]["leaf"], union) and np.array_equal(got[1]["leaf"], union)
    assert bool(got[0]["top"][0, 0]) and got[0]["top"].shape == (1, 1)
    lv1 = part.levels[1]
    leaves = part.leaves
    for a, sa in enumerate(lv1):
        for b, sb in enumerate(lv1):
            ra = [k for k, s in enumerate(leaves) if sa.fn_lo <= s.fn_lo and s.fn_hi <= sa.fn_hi]
            rb = [k for k, s in enumerate(leaves) if sb.fn_lo <= s.fn_lo and s.fn_hi <= sb.fn_hi]
            assert bool(got[0]["l1"][a, b]) == bool(union[np.ix_(ra, rb)].any())
    assert 0 < int(got[0]["nnz"]) < nl * nl                        # the band leaves tiles out
    assert int(got[0]["packed"]) == int(got[0]["stored"])
    assert int(got[0]["owned"]) + int(got[1]["owned"]) == 8 * int(got[0]["packed"])
