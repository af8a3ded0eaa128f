"""Multi-GPU exchange build: product-tree sharding + NCCL reduction of K.

SURVEY.md 8(e): subtrees of the product (hextree) task space are independent
except for accumulation into K (the reference's depth-1 thread farm,
exchange_naive.py:220-235, and the paper's parallel argument).  Every rank
expands the top levels identically to a cut level whose frontier holds
>= 1024 tasks per rank, takes the tasks a fixed hash of the task index
assigns to it (deterministic; cyclic or contiguous selections optional), runs traversal + leaf screening + ERIs on it into a
private K, and the partial K are summed with one all-reduce (NCCL over
NVLink; gloo on CPU for the host-logic tests).  The fourfold epilogue
(symmetrize_final) runs once on the reduced K.  Counters are summed the same
way; work above the cut is counted by shard 0 only.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .exchange import CASE_LABELS, SymmetryCounters, TraversalCounters, run_exchange


def split_by_cost(costs, world: int):
    """Contiguous ranges [b, e) of a frontier with ~equal summed cost per rank."""
    costs = np.asarray(costs, dtype=float)
    n = len(costs)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    cum = np.concatenate([[0.0], np.cumsum(costs)])
    total = cum[-1]
    cuts = [0]
    for r in range(1, world):
        cuts.append(int(np.searchsorted(cum, total * r / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.minimum(cuts, n))
    return [(int(cuts[r]), int(cuts[r + 1])) for r in range(world)]


def frontier(bra, ket, P, tau_2e, mode, symmetry, level):
    """Expand-list size (and per-task cost estimates) at `level`."""
    n = ctypes.c_int64(0)
    sym = 2 if symmetry == "eightfold" else (1 if symmetry else 0)
    _native.check(_native.lib().hxf_frontier(bra._t.handle, ket._t.handle, P._t.handle, float(tau_2e),
                                             0 if mode == "schwarz" else 1, sym,
                                             int(level), ctypes.byref(n), None, 0,
                                             _native.current_stream()))
    count = int(n.value)
    costs = np.empty(max(count, 1))
    _native.check(_native.lib().hxf_frontier(bra._t.handle, ket._t.handle, P._t.handle, float(tau_2e),
                                             0 if mode == "schwarz" else 1, sym,
                                             int(level), ctypes.byref(n), _native.ptr(costs), count,
                                             _native.current_stream()))
    return count, costs[:count]


def split_cyclic(n: int, world: int):
    """Rank r takes frontier tasks r, r + world, r + 2 world, ... as (begin, end, stride).

    Frontier order follows the space-filling shell order, so neighbouring tasks
    have similar cost; dealing them out cyclically balances ranks without a
    per-task cost model (contiguous ranges of a 3D cluster's frontier differ by
    the density of surviving work in their region)."""
    return [(min(r, n), n, max(world, 1)) for r in range(max(world, 1))]


def _splitmix64(x):
    z = (np.asarray(x, dtype=np.uint64) + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def split_hashed(n: int, world: int, seed: int = 0x1401_6961):
    """Rank of task t = SplitMix64(t + seed) mod world, as per-rank uint8 masks.

    The frontier has periodic structure (the 16 children of a parent differ
    systematically: bra/ket children on the block diagonal carry most of the
    surviving work), which a stride-`world` deal aliases with; a hash breaks
    the period, and a deep cut (many tasks per rank) averages the rest."""
    owner = _owner(n, world, seed)
    return [(0 if r == 0 else 1, n, (owner == r).astype(np.uint8)) for r in range(max(world, 1))]


# Seconds per unit of counted work on one B200 (c5 fourfold stage times / counters:
# ERI 5.0 s / 2.16e10 surviving quartets, leaf screen 2.66 s / 9.75e8 leaf tasks,
# traversal 0.26 s / 5.64e9 visited tasks); only their ratios matter.
COST_PER_QUARTET, COST_PER_LEAF_TASK, COST_PER_VISIT = 2.32e-10, 2.73e-9, 4.6e-11


def group_costs(bra, ket, P, tau_2e, mode, symmetry, level, n, groups, K_scratch, group=None):
    """Modelled cost of each hashed task group of the level-`level` frontier (n tasks).

    One counters-only build (evaluate = 0: traversal + leaf screen, no ERIs) per
    group; cost = the counted surviving quartets, leaf tasks and visits weighted by
    their measured unit times.  Under torch.distributed every rank measures every
    world-th group and the cost vector is all-reduced (same result on every rank).
    K_scratch: a device float64 n_fn x n_fn tensor the counting builds may clear."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    owner = _owner(n, groups)
    cost = np.zeros(groups)
    for g in range(rank, groups, world):
        mask = (owner == g).astype(np.uint8)
        if not mask.any():
            continue
        _, c, _ = run_exchange(bra, ket, P, tau_2e, mode, symmetry, False, None, K_out=K_scratch,
                               shard=(level, 1, n, mask), symmetrize=False)
        cost[g] = (COST_PER_QUARTET * c.eri_shell_quartets + COST_PER_LEAF_TASK * c.leaf_contractions
                   + COST_PER_VISIT * c.tasks_visited)
    if world > 1:
        t = torch.from_numpy(cost).to(K_scratch.device)
        dist.all_reduce(t, group=group)
        cost = t.cpu().numpy()
    return cost


def _owner(n, buckets, seed=0x1401_6961):
    with np.errstate(over="ignore"):
        return (_splitmix64(np.arange(n, dtype=np.uint64) + np.uint64(seed))
                % np.uint64(max(buckets, 1))).astype(np.int64)


def split_lpt(n, world, groups, costs):
    """Assign hashed task groups to ranks by longest-processing-time-first (ties by
    group index, so deterministic); returns per-rank (begin, n, mask) like split_hashed."""
    load = np.zeros(max(world, 1))
    rank_of = np.zeros(groups, dtype=np.int64)
    for g in sorted(range(groups), key=lambda g: (-costs[g], g)):
        r = int(np.argmin(load))
        rank_of[g] = r
        load[r] += costs[g]
    owner = rank_of[_owner(n, groups)] if n else np.zeros(0, dtype=np.int64)
    return [(0 if r == 0 else 1, n, (owner == r).astype(np.uint8)) for r in range(max(world, 1))]


def plan(bra, ket, P, tau_2e, mode, symmetry, world, min_tasks_per_rank=None, strategy="hashed",
         K_scratch=None, groups_per_rank=16, group=None):
    """Choose the cut level and this job's shard selections (same on every rank).

    Returns (level, [(begin, end, stride_or_mask)] per rank) for
    run_exchange(shard=(level,) + selection).  Strategies: "hashed"
    (split_hashed at a cut with >= 1024 tasks per rank; default), "balanced"
    (hashed groups_per_rank * world task groups, costs measured by counters-only
    builds, LPT-assigned; needs K_scratch), "cyclic" (split_cyclic, >= 64 per
    rank) or "contiguous" (split_by_cost ranges)."""
    if strategy not in ("hashed", "balanced", "cyclic", "contiguous"):
        raise ValueError(f"unknown shard strategy {strategy!r}")
    if min_tasks_per_rank is None:
        min_tasks_per_rank = 1024 if strategy in ("hashed", "balanced") else 64
    n_levels = len(bra._t.ds.levels)
    level, count, costs = 0, 1, np.ones(1)
    for L in range(n_levels - 1):
        count, costs = frontier(bra, ket, P, tau_2e, mode, symmetry, L)
        level = L
        if count >= min_tasks_per_rank * world:
            break
    if strategy == "hashed":
        return level, split_hashed(count, world)
    if strategy == "balanced":
        if world <= 1:
            return level, split_hashed(count, world)
        if K_scratch is None:
            raise ValueError("the balanced plan needs K_scratch (device n_fn x n_fn float64)")
        groups = groups_per_rank * world
        costs = group_costs(bra, ket, P, tau_2e, mode, symmetry, level, count, groups, K_scratch, group)
        return level, split_lpt(count, world, groups, costs)
    if strategy == "cyclic":
        return level, split_cyclic(count, world)
    return level, [(b, e, 1) for b, e in split_by_cost(costs, world)]


def counters_vector(c) -> np.ndarray:
    """Flatten an hxf counters struct to float64 (int64 counts are exact below 2^53)."""
    v = [c.tasks_visited, c.tasks_culled_screening, c.tasks_culled_absent, c.leaf_contractions,
         c.eri_shell_quartets, c.quartets_culled_leaf, c.tasks_expanded, c.children_spawned,
         c.links_culled_screening, c.links_culled_absent, c.ties_task, c.ties_leaf,
         c.prim_quartets]
    v += list(c.case_tasks) + list(c.case_leaf_tasks)
    v += list(c.class_quartets) + list(c.class_prim_quartets)
    v.append(c.culled_bound_ledger)
    return np.asarray(v, dtype=np.float64)


def counters_from_vector(v, symmetric):
    out = SymmetryCounters() if symmetric else TraversalCounters()
    keys = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent", "leaf_contractions",
            "eri_shell_quartets", "quartets_culled_leaf", "tasks_expanded", "children_spawned")
    for k, x in zip(keys, v[:8]):
        setattr(out, k, int(round(x)))
    if symmetric:
        out.links_culled_screening = int(round(v[8]))
        out.links_culled_absent = int(round(v[9]))
        for g, lab in enumerate(CASE_LABELS):
            out.case_tasks[lab] = int(round(v[13 + g]))
            out.case_leaf_tasks[lab] = int(round(v[22 + g]))
    out.ties_task, out.ties_leaf, out.prim_quartets = (int(round(x)) for x in v[10:13])
    out.culled_bound_ledger = float(v[-1])
    return out


def allreduce_partials(K, counters_vec, group=None):
    """Sum partial K and counter vectors over the job (NCCL on GPU, gloo on CPU)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(K, group=group)
        dist.all_reduce(counters_vec, group=group)
    return K, counters_vec


class _NativeBlockOps:
    """Block-sparse tile ops of libhxf (csrc/reduce.cu) on CUDA int64 tensors."""

    @staticmethod
    def _check(K):
        from .exchange import check_device_matrix
        check_device_matrix(K, K.shape[0] if K.dim() == 2 else -1, "int64", None, "K")

    @staticmethod
    def mask(K, bs):
        import torch
        _NativeBlockOps._check(K)
        n = K.shape[0]
        nb = (n + bs - 1) // bs
        m = torch.empty(nb * nb, dtype=torch.uint8, device=K.device)
        _native.check(_native.lib().hxf_block_mask(ctypes.c_void_p(K.data_ptr()), n, bs,
                                                   ctypes.c_void_p(m.data_ptr()), _native.current_stream()))
        return m

    @staticmethod
    def slots(m):
        import torch
        slot = torch.empty(m.numel() + 1, dtype=torch.int64, device=m.device)
        cnt = ctypes.c_int64(0)
        _native.check(_native.lib().hxf_block_slots(ctypes.c_void_p(m.data_ptr()), m.numel(),
                                                    ctypes.c_void_p(slot.data_ptr()), ctypes.byref(cnt),
                                                    _native.current_stream()))
        return slot, int(cnt.value)

    @staticmethod
    def pack(K, bs, m, slot, nblk):
        import torch
        _NativeBlockOps._check(K)
        buf = torch.empty(max(1, nblk) * bs * bs, dtype=torch.int64, device=K.device)
        _native.check(_native.lib().hxf_block_pack(ctypes.c_void_p(K.data_ptr()), K.shape[0], bs,
                                                   ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(slot.data_ptr()),
                                                   ctypes.c_void_p(buf.data_ptr()), _native.current_stream()))
        return buf

    @staticmethod
    def unpack(K, bs, m, slot, buf):
        _NativeBlockOps._check(K)
        _native.check(_native.lib().hxf_block_unpack(ctypes.c_void_p(K.data_ptr()), K.shape[0], bs,
                                                     ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(slot.data_ptr()),
                                                     ctypes.c_void_p(buf.data_ptr()), _native.current_stream()))


def allreduce_fixed_sparse(Kfx, counters_vec, group=None, block=64, ops=None):
    """Block-sparse exact all-reduce of int64 fixed-point shard accumulators
    (SURVEY §8(f) f4): OR of the per-rank nonzero-tile masks (uint8 max), then an
    int64 sum of only the union's tiles.  A tile no rank flags is zero everywhere,
    so the result is bitwise the dense all-reduce.  Returns (Kfx, counters_vec,
    stats) with the tile count and the bytes each rank contributed."""
    import torch.distributed as dist
    ops = ops or _NativeBlockOps
    m = ops.mask(Kfx, block)
    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    if multi:
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(counters_vec, group=group)
    slot, nblk = ops.slots(m)
    if multi and nblk:
        buf = ops.pack(Kfx, block, m, slot, nblk)
        dist.all_reduce(buf, group=group)
        ops.unpack(Kfx, block, m, slot, buf)
    n = Kfx.shape[0]
    stats = {"block": block, "tiles": int(m.numel()), "tiles_nonzero": nblk,
             "bytes_sparse": nblk * block * block * 8 + int(m.numel()), "bytes_dense": n * n * 8}
    return Kfx, counters_vec, stats


# ---------------------------------------------------------------------------
# K as a block-sparse quadtree over the partition + a row-owning reduce-scatter
# (second part; PAPER.md:174-198 writes the K update block by block over
# the same index bisection as P).

def leaf_function_ranges(part):
    """(flo, fhi): int32 function ranges of the partition's leaf spans, in order."""
    leaves = part.leaves
    return (np.asarray([s.fn_lo for s in leaves], dtype=np.int32),
            np.asarray([s.fn_hi for s in leaves], dtype=np.int32))


class KQuadtree:
    """Occupancy quadtree of a block-sparse K: level L holds one flag per (row span,
    column span) pair of the partition's level-L spans (Partition.levels: ragged leaves
    repeat at deeper levels), set when any leaf tile below it holds a nonzero.  The
    bottom level is the leaf-tile mask the device computed (hxf_span_mask)."""

    def __init__(self, part, leaf_mask):
        leaves = part.leaves
        nl = len(leaves)
        m = np.asarray(leaf_mask, dtype=np.uint8).reshape(nl, nl)
        self.partition = part
        self.leaf_mask = m
        self.flo, self.fhi = leaf_function_ranges(part)
        first = {id(s): k for k, s in enumerate(leaves)}
        # leaf-index range [a, b) under every span of every level
        def rng(s):
            t = s
            while not t.is_leaf:
                t = t.left
            a = first[id(t)]
            t = s
            while not t.is_leaf:
                t = t.right
            return a, first[id(t)] + 1
        integ = np.zeros((nl + 1, nl + 1), dtype=np.int64)
        integ[1:, 1:] = m.astype(np.int64).cumsum(0).cumsum(1)
        self.levels = []
        for spans in part.levels:
            r = np.asarray([rng(s) for s in spans], dtype=np.int64)
            a, b = r[:, 0], r[:, 1]
            cnt = integ[b][:, b] - integ[a][:, b] - integ[b][:, a] + integ[a][:, a]
            self.levels.append(cnt > 0)

    @property
    def n_levels(self):
        return len(self.levels)

    def occupied(self, level, i, j):
        return bool(self.levels[level][i, j])

    @property
    def nnz_tiles(self):
        return int(self.leaf_mask.sum())

    @property
    def stored_elements(self):
        nf = (self.fhi - self.flo).astype(np.int64)
        return int((self.leaf_mask.astype(np.int64) * np.outer(nf, nf)).sum())

    def fill(self, level=None):
        """Occupied fraction of a level's nodes (default: the leaf level)."""
        lv = self.levels[-1 if level is None else level]
        return float(lv.mean()) if lv.size else 0.0


class _NativeSpanOps:
    """Leaf-span tile ops of libhxf (csrc/reduce.cu) on CUDA int64 tensors."""

    @staticmethod
    def mask(K, flo_d, fhi_d):
        import torch
        nl = flo_d.numel()
        m = torch.empty(nl * nl, dtype=torch.uint8, device=K.device)
        _native.check(_native.lib().hxf_span_mask(ctypes.c_void_p(K.data_ptr()), K.shape[1],
                                                  ctypes.c_void_p(flo_d.data_ptr()), ctypes.c_void_p(fhi_d.data_ptr()),
                                                  nl, ctypes.c_void_p(m.data_ptr()), _native.current_stream()))
        return m

    @staticmethod
    def move(K, row_base, flo_d, fhi_d, r0, r1, m, off, off_base, buf, pack):
        fn = _native.lib().hxf_span_pack if pack else _native.lib().hxf_span_unpack
        _native.check(fn(ctypes.c_void_p(K.data_ptr()), K.shape[1], int(row_base),
                         ctypes.c_void_p(flo_d.data_ptr()), ctypes.c_void_p(fhi_d.data_ptr()), flo_d.numel(),
                         int(r0), int(r1), ctypes.c_void_p(m.data_ptr()), ctypes.c_void_p(off.data_ptr()),
                         int(off_base), ctypes.c_void_p(buf.data_ptr()), _native.current_stream()))

    @staticmethod
    def fold(K):
        _native.check(_native.lib().hxf_fixed_fold(ctypes.c_void_p(K.data_ptr()), K.shape[0],
                                                   _native.current_stream()))


class KRowBlock:
    """What one rank holds after reduce_scatter_quadtree: the reduced leaf tiles of its
    row spans [r0, r1) (functions [f0, f1)), packed, in fixed point."""

    def __init__(self, r0, r1, f0, f1, n, flo_d, fhi_d, mask, off, off_base, buf, scale, folded, ops):
        self.r0, self.r1, self.f0, self.f1, self.n = r0, r1, f0, f1, n
        self._flo, self._fhi, self.mask, self.off, self.off_base = flo_d, fhi_d, mask, off, off_base
        self.tiles = buf
        self.scale, self.folded, self._ops = scale, folded, ops

    def dense_fixed(self):
        """(f1 - f0) x n int64 row block (zero outside the stored tiles)."""
        import torch
        out = torch.zeros((max(self.f1 - self.f0, 0), self.n), dtype=torch.int64, device=self.tiles.device)
        if self.r1 > self.r0 and out.numel():
            self._ops.move(out, self.f0, self._flo, self._fhi, self.r0, self.r1, self.mask, self.off,
                           self.off_base, self.tiles, False)
        return out

    def dense(self):
        """The rank's rows of K in FP64: fixed / 2^scale, halved when the partials were folded
        (K = (A + A^T) / 2, the fourfold epilogue of exchange_symmetry.py:197-209)."""
        import torch
        k = torch.ldexp(self.dense_fixed().to(torch.float64),
                        torch.tensor(-self.scale - (1 if self.folded else 0), device=self.tiles.device))
        return k


def reduce_scatter_quadtree(Kfx, part, scale, group=None, fold=False, ops=None):
    """Row-owning block-sparse reduction of the shard accumulators.

    Kfx: this rank's n x n int64 fixed-point partial.  fold=True first forms A + A^T in
    place (exact), so the reduced rows are already those of the symmetrised fourfold K.
    The leaf-tile occupancy is OR-ed over the job, the union's tiles are packed in tile
    row-major order, the row spans are cut into one contiguous range per rank with about
    equal packed elements, and each range is sum-reduced to its owner (one reduce per
    owner: NCCL and gloo both carry it; the bytes are those of a reduce-scatter).  No
    rank receives rows it does not own and no zero tile travels.  Returns (KRowBlock,
    KQuadtree, stats)."""
    import torch
    import torch.distributed as dist
    ops = ops or _NativeSpanOps
    multi = dist.is_initialized() and dist.get_world_size(group) > 1
    world = dist.get_world_size(group) if multi else 1
    rank = dist.get_rank(group) if multi else 0
    n = Kfx.shape[0]
    flo, fhi = leaf_function_ranges(part)
    nl = len(flo)
    flo_d = torch.from_numpy(flo).to(Kfx.device)
    fhi_d = torch.from_numpy(fhi).to(Kfx.device)
    if fold:
        ops.fold(Kfx)
    m = ops.mask(Kfx, flo_d, fhi_d)
    if multi:
        dist.all_reduce(m, op=dist.ReduceOp.MAX, group=group)
    nf = (fhi_d - flo_d).to(torch.int64)
    sizes = (m.view(nl, nl).to(torch.int64) * nf[:, None] * nf[None, :]).reshape(-1)
    off = torch.zeros(nl * nl + 1, dtype=torch.int64, device=Kfx.device)
    torch.cumsum(sizes, 0, out=off[1:])
    row_start = off[::nl][: nl + 1].cpu().numpy() if nl else np.zeros(1, dtype=np.int64)
    if len(row_start) < nl + 1:
        row_start = np.append(row_start, int(off[-1]))
    total = int(row_start[-1])
    # row-span cuts: rank k owns spans [cut[k], cut[k+1]) holding ~total / world elements
    cut = [0]
    for k in range(1, world):
        cut.append(int(np.searchsorted(row_start, total * k / world, side="left")))
    cut.append(nl)
    cut = np.maximum.accumulate(np.minimum(cut, nl))
    buf = torch.empty(max(total, 1), dtype=torch.int64, device=Kfx.device)
    if total:
        ops.move(Kfx, 0, flo_d, fhi_d, 0, nl, m, off, 0, buf, True)
    mine = None
    works = []
    for k in range(world):
        a, b = int(row_start[cut[k]]), int(row_start[cut[k + 1]])
        seg = buf[a:b]
        if multi and b > a:
            works.append(dist.reduce(seg, dst=dist.get_global_rank(group, k) if group is not None else k,
                                     group=group, async_op=True))
        if k == rank:
            mine = (int(cut[k]), int(cut[k + 1]), a, b)
    for w in works:
        w.wait()
    r0, r1, a, b = mine
    f0 = int(flo[r0]) if r1 > r0 else 0
    f1 = int(fhi[r1 - 1]) if r1 > r0 else 0
    block = KRowBlock(r0, r1, f0, f1, n, flo_d, fhi_d, m, off, a, buf[a:b].clone(), scale, fold, ops)
    tree = KQuadtree(part, m.cpu().numpy())
    stats = {"leaf_tiles": nl * nl, "leaf_tiles_nonzero": tree.nnz_tiles, "packed_elements": total,
             "bytes_packed": total * 8, "bytes_dense": n * n * 8, "bytes_owned": (b - a) * 8,
             "row_spans": (r0, r1), "rows": (f0, f1)}
    return block, tree, stats


def exchange_sharded(bra, ket, P, tau_2e, mode, symmetry, K_dev, group=None, shards=None,
                     sparse_block=None):
    """One rank's share of a sharded build + the all-reduce of K and counters.

    K_dev: torch CUDA tensor (n x n float64), overwritten with the full K on
    every rank.  Each shard's K is its 64-bit fixed-point accumulator (same
    scale on every rank); the int64 all-reduce is an exact integer sum, so the
    reduced K is bitwise the single-device K.  sparse_block=bs all-reduces only
    the bs x bs tiles some rank holds a nonzero in (allreduce_fixed_sparse; same
    K bit for bit).  Returns (counters, shard plan).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if shards is None:
        shards = plan(bra, ket, P, tau_2e, mode, symmetry, world)
    level, ranges = shards
    b, e, stride = ranges[rank]
    from .exchange import check_device_matrix
    check_device_matrix(K_dev, bra.row.n_functions, "float64", bra._t.ds.device_index, "K_dev")
    Kfx = K_dev.view(torch.int64)          # the FP64 buffer reused for the accumulator
    (_, S), c, _ = run_exchange(bra, ket, P, tau_2e, mode, symmetry, True, None, K_out=Kfx,
                                shard=(level, b, e, stride), symmetrize=False,
                                K_fixed=True)
    vec = torch.from_numpy(counters_vector(c)).to(K_dev.device)
    if sparse_block:
        allreduce_fixed_sparse(Kfx, vec, group, block=int(sparse_block))
    else:
        allreduce_partials(Kfx, vec, group)
    _native.check(_native.lib().hxf_fixed_to_double(ctypes.c_void_p(Kfx.data_ptr()), Kfx.numel(), S,
                                                    ctypes.c_void_p(K_dev.data_ptr()),
                                                    _native.current_stream()))
    if symmetry is True:  # fourfold; the eightfold K (A + A^T) is symmetric by construction
        _native.check(_native.lib().hxf_symmetrize(ctypes.c_void_p(K_dev.data_ptr()), K_dev.shape[0],
                                                   1e-10, _native.current_stream()))
    return counters_from_vector(vec.cpu().numpy(), symmetry), shards


def exchange_sharded_rows(bra, ket, P, tau_2e, mode, symmetry, K_dev, group=None, shards=None):
    """One rank's share of a sharded build, reduced with reduce_scatter_quadtree: every rank
    ends with only its own rows of K (a KRowBlock of leaf tiles) and the K quadtree.

    K_dev (n x n float64, CUDA) is the rank's scratch for its fixed-point partial.  For the
    fourfold driver the partials are folded (A + A^T, exact) before the reduction, so the
    owned rows are those of the symmetrised K = (A + A^T) / 2 (exchange_symmetry.py:197-209);
    the 1e-10 asymmetry check of that epilogue needs both triangles of the reduced matrix and
    is not made here.  Returns (KRowBlock, KQuadtree, counters, stats)."""
    import torch
    import torch.distributed as dist

    if symmetry not in (False, True):
        raise ValueError("exchange_sharded_rows: naive or fourfold driver")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if shards is None:
        shards = plan(bra, ket, P, tau_2e, mode, symmetry, world)
    level, ranges = shards
    b, e, stride = ranges[rank]
    from .exchange import check_device_matrix
    check_device_matrix(K_dev, bra.row.n_functions, "float64", bra._t.ds.device_index, "K_dev")
    Kfx = K_dev.view(torch.int64)
    (_, S), c, _ = run_exchange(bra, ket, P, tau_2e, mode, symmetry, True, None, K_out=Kfx,
                                shard=(level, b, e, stride), symmetrize=False, K_fixed=True)
    vec = torch.from_numpy(counters_vector(c)).to(K_dev.device)
    if dist.is_initialized() and world > 1:
        dist.all_reduce(vec, group=group)
    block, tree, stats = reduce_scatter_quadtree(Kfx, bra._t.partition,
                                                 S, group=group, fold=bool(symmetry))
    return block, tree, counters_from_vector(vec.cpu().numpy(), symmetry), stats
