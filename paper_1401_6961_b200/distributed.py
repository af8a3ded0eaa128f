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
