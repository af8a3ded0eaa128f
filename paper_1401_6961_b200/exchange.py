"""Drop-in exchange drivers: the reference's entry points over libhxf.

  build_exchange_naive ...... exchange_naive.py:200-240
  build_exchange_symmetric .. exchange_symmetry.py:364-409
  TraversalCounters ......... exchange_naive.py:28-65
  SymmetryCounters .......... exchange_symmetry.py:72-132
  screening_test / culled_task_bound / classify_quartet / symmetrize_final:
                              scalar host helpers with the reference semantics
                              (exchange_naive.py:68-108, exchange_symmetry.py:135-209)

Same signatures, return types and exceptions as the reference.  The whole
build (traversal, leaf screening, ERIs, contraction, symmetrisation) runs in
hxf_exchange on the GPU; ``threads`` is accepted for API compatibility (the
device build is deterministic for any value).  ``quartet_log`` receives the
evaluated shell quartets in lexicographic order (the reference appends in
depth-first order; its tests compare sets and lengths).
"""

from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from ._native import LogicError
from .basis import InvalidArgumentError
from .quadtree import MatrixQuadtree, ShellPairNode

CASE_LABELS = ("A", "B", "C", "D", "E", "F1", "F2", "H", "SPARSE")

_SLOT_TABLE = (
    ("K[mu,sig]", "P[nu,lam]", "1"),
    ("K[nu,sig]", "P[mu,lam]", "[mu!=nu]"),
    ("K[mu,lam]", "P[nu,sig]", "[lam!=sig]"),
    ("K[nu,lam]", "P[mu,sig]", "[mu!=nu][lam!=sig]"),
)
_SLOT_TRANSPOSES = ((False, False), (True, False), (False, True), (True, True))


@dataclass
class TraversalCounters:
    tasks_visited: int = 0
    tasks_culled_screening: int = 0
    tasks_culled_absent: int = 0
    leaf_contractions: int = 0
    eri_shell_quartets: int = 0
    quartets_culled_leaf: int = 0
    tasks_expanded: int = 0
    children_spawned: int = 0
    culled_bound_ledger: float = 0.0
    # device extras (not part of the reference's to_dict)
    ties_task: int = 0
    ties_leaf: int = 0
    screen_bytes: int = 0   # leaf screen: SURVEY 8(d) algorithmic bytes (bench roofline)
    prim_quartets: int = 0

    _KEYS = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
             "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
             "tasks_expanded", "children_spawned", "culled_bound_ledger")

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in self._KEYS}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)

    def merge(self, other) -> None:
        for k in self._KEYS + ("ties_task", "ties_leaf", "prim_quartets"):
            setattr(self, k, getattr(self, k) + getattr(other, k))


@dataclass
class SymmetryCounters:
    tasks_visited: int = 0
    tasks_culled_screening: int = 0
    tasks_culled_absent: int = 0
    leaf_contractions: int = 0
    eri_shell_quartets: int = 0
    quartets_culled_leaf: int = 0
    tasks_expanded: int = 0
    children_spawned: int = 0
    links_culled_screening: int = 0
    links_culled_absent: int = 0
    culled_bound_ledger: float = 0.0
    case_tasks: dict = field(default_factory=lambda: {c: 0 for c in CASE_LABELS})
    case_leaf_tasks: dict = field(default_factory=lambda: {c: 0 for c in CASE_LABELS})
    ties_task: int = 0
    ties_leaf: int = 0
    screen_bytes: int = 0   # leaf screen: SURVEY 8(d) algorithmic bytes (bench roofline)
    prim_quartets: int = 0

    _KEYS = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
             "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
             "tasks_expanded", "children_spawned", "links_culled_screening",
             "links_culled_absent", "culled_bound_ledger")

    def to_dict(self) -> dict:
        d = {k: getattr(self, k) for k in self._KEYS}
        d["case_tasks"] = dict(self.case_tasks)
        d["case_leaf_tasks"] = dict(self.case_leaf_tasks)
        return d

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)

    def case_breakdown_csv(self, leaf_only: bool = False) -> str:
        counts = self.case_leaf_tasks if leaf_only else self.case_tasks
        total = sum(counts.values())
        lines = ["case,count,percent"]
        for label in CASE_LABELS:
            pct = 100.0 * counts[label] / total if total else 0.0
            lines.append(f"{label},{counts[label]},{pct:.4f}")
        return "\n".join(lines) + "\n"

    def merge(self, other) -> None:
        for k in self._KEYS + ("ties_task", "ties_leaf", "prim_quartets"):
            setattr(self, k, getattr(self, k) + getattr(other, k))
        for c in CASE_LABELS:
            self.case_tasks[c] += other.case_tasks[c]
            self.case_leaf_tasks[c] += other.case_leaf_tasks[c]


def _sorted_product(a, b, c):
    lo, mid, hi = sorted((a, b, c))
    return lo * mid * hi


def screening_test(bra_norm, p_norm, ket_norm, tau_2e, mode="schwarz") -> bool:
    """True when the blocked Almlof-Ahlrichs bound culls the task (exchange_naive.py:74-88)."""
    if bra_norm < 0.0 or p_norm < 0.0 or ket_norm < 0.0:
        raise InvalidArgumentError("screening norms must be non-negative")
    if mode == "schwarz":
        bra_norm, ket_norm = math.sqrt(bra_norm), math.sqrt(ket_norm)
    elif mode != "literal":
        raise InvalidArgumentError(f"unknown screening mode {mode!r}")
    return _sorted_product(bra_norm, p_norm, ket_norm) <= tau_2e


def culled_task_bound(bra, p_norm, ket, transpose_bra=False, transpose_ket=False) -> float:
    """Rigorous max-abs bound on one culled task's K contribution (exchange_naive.py:91-102)."""
    bs = bra.colsum_max if transpose_bra else bra.rowsum_max
    ks = ket.rowsum_max if transpose_ket else ket.colsum_max
    return 0.5 * p_norm * math.sqrt(max(bs, 0.0)) * math.sqrt(max(ks, 0.0))


@dataclass(frozen=True)
class SlotSpec:
    sink: str
    source: str
    weight: str
    valid: bool = True


@dataclass
class SymmetryCase:
    case_id: str
    slots: tuple


def _same_node(b, k) -> bool:
    if b is k:
        return True
    return (isinstance(b, ShellPairNode) and isinstance(k, ShellPairNode) and b._t is k._t
            and (b._level, b._r, b._c) == (k._level, k._r, k._c))


def _case_label(b, k) -> str:
    mu, nu, lam, sig = b.row, b.col, k.row, k.col
    if _same_node(b, k):
        return "E"
    bd, kd = mu is nu, lam is sig
    if bd and kd:
        return "H"
    if bd or kd:
        return "B"
    if nu is lam or mu is sig:
        return "A"
    if mu is lam:
        return "F1"
    if nu is sig:
        return "F2"
    if nu.fn_lo < lam.fn_lo or sig.fn_lo < mu.fn_lo:
        return "A"
    if (lam.fn_lo < mu.fn_lo) != (sig.fn_lo < nu.fn_lo):
        return "C"
    return "D"


def classify_quartet(bra, ket, present=(True, True, True, True)) -> SymmetryCase:
    """Span-relation case of one canonical task (exchange_symmetry.py:176-194)."""
    if bra.row.fn_lo > bra.col.fn_lo or ket.row.fn_lo > ket.col.fn_lo:
        raise LogicError("non-canonical task: pair spans out of order")
    present = tuple(bool(v) for v in present)
    label = _case_label(bra, ket)
    if not all(present):
        label = "SPARSE"
    slots = tuple(SlotSpec(s, src, w, valid=present[g])
                  for g, (s, src, w) in enumerate(_SLOT_TABLE))
    return SymmetryCase(case_id=label, slots=slots)


def symmetrize_final(K_raw, tol: float = 1e-10) -> np.ndarray:
    """(K + K^T)/2 after an asymmetry check (exchange_symmetry.py:197-209).

    Host utility for callers; the device build symmetrises on the GPU.
    """
    K_raw = np.asarray(K_raw, dtype=float)
    asym = float(np.abs(K_raw - K_raw.T).max()) if K_raw.size else 0.0
    if asym > tol:
        raise LogicError(f"asymmetry {asym:.3e} exceeds {tol:.1e}; symmetry update set is inconsistent")
    return 0.5 * (K_raw + K_raw.T)


def _check_same_partition(bra, ket, p):
    roots = {id(bra.row), id(bra.col), id(ket.row), id(ket.col), id(p.row), id(p.col)}
    if len(roots) != 1:
        raise InvalidArgumentError("bra, ket and P must be built over the same partition")


def check_device_matrix(K, n, dtype, device=None, what="K_out"):
    """A device output buffer must be a contiguous CUDA (n, n) tensor of `dtype`
    on the system's device: the library writes n*n elements through its pointer."""
    if not (hasattr(K, "is_cuda") and K.is_cuda):
        raise InvalidArgumentError(f"{what} must be a CUDA tensor")
    if tuple(K.shape) != (n, n):
        raise InvalidArgumentError(f"{what} must have shape ({n}, {n}), got {tuple(K.shape)}")
    if str(K.dtype) != f"torch.{dtype}":
        raise InvalidArgumentError(f"{what} must be {dtype}, got {K.dtype}")
    if not K.is_contiguous():
        raise InvalidArgumentError(f"{what} must be contiguous")
    if device is not None and K.device.index != device:
        raise InvalidArgumentError(f"{what} is on cuda:{K.device.index}, the system on cuda:{device}")


def _require_root(node, what):
    if node._level != 0:
        raise InvalidArgumentError(f"{what}: the device drivers start from the tree root")


def _start_node(bra, ket, P):
    """(level, index) of the diagonal start node.  The reference accepts any
    bra/ket/P whose six spans are one Span object (_check_same_partition,
    exchange_naive.py:105-108): the root or a diagonal subtree (r, r).  A ragged
    leaf repeats at deeper levels; every view of it denotes the same node."""
    nodes = (bra, ket, P)
    for nd in nodes:
        if nd._r != nd._c:
            raise InvalidArgumentError("bra, ket and P must be built over the same partition")
    lv = min(nd._level for nd in nodes)
    idx = bra._t.ds.index[lv][id(bra.row)]
    return lv, idx


def run_exchange(bra, ket, P, tau_2e, mode, symmetry, evaluate=True, quartet_log=None,
                 K_out=None, shard=None, symmetrize=True, digest=None, digest_sample=(1, 0),
                 K_fixed=False, tie_log=None, screen_bytes=False):
    """Low-level call of hxf_exchange.

    K_out: None (return a new host array), or a CUDA tensor (n x n float64)
    written in place on the device.  shard: None, (level, begin, end) or
    (level, begin, end, stride) (every stride-th frontier task of [begin, end)) or
    (level, begin, n, mask) (frontier tasks t with mask[t] != 0, numpy uint8[n];
    work above the cut is counted when begin == 0).
    K_fixed: K_out (a CUDA int64 n x n tensor) receives the 64-bit fixed-point
    accumulator and the returned K is (K_out, S) with value = K_out * 2^-S
    (exact integer sums across shards; include/hxf.h).
    digest: None, or a caller-owned numpy uint64[3] filled with the
    order-independent digest (count, sum h, sum h(h)) of the evaluated quartet
    tuples with i % digest_sample[0] == digest_sample[1] (include/hxf.h).
    tie_log: None, or a list extended with one dict per culling comparison of the
    task and leaf stages whose bound lies within 1e-12 relative of tau_2e (stage,
    level, slot, decision, ids, bound, threshold, contribution: include/hxf.h
    hxf_tie_record; at most TIE_CAPACITY records, the counters hold the totals).
    Returns (K or None, hxf counters struct, list of logged quartets or None).
    """
    if not (tau_2e >= 0.0):
        raise InvalidArgumentError("tau_2e must be non-negative")
    if mode not in ("schwarz", "literal"):
        raise InvalidArgumentError(f"unknown screening mode {mode!r}")
    _check_same_partition(bra, ket, P)
    root_level, root_index = _start_node(bra, ket, P)
    L = _native.lib()
    n = bra.row.n_functions
    opts = _native.ExchangeOpts()
    opts.root_level, opts.root_index = root_level, root_index
    opts.tau_2e = float(tau_2e)
    opts.mode = 0 if mode == "schwarz" else 1
    # symmetry: False / True (fourfold) / "eightfold"
    opts.symmetry = 2 if symmetry == "eightfold" else (1 if symmetry else 0)
    opts.evaluate = 1 if evaluate else 0
    opts.symmetrize = 1 if symmetrize else 0
    if shard is None:
        opts.shard_level, opts.shard_begin, opts.shard_end = -1, 0, 0
    else:
        opts.shard_level, opts.shard_begin, opts.shard_end = (int(x) for x in shard[:3])
        sel = shard[3] if len(shard) > 3 else 1
        if isinstance(sel, np.ndarray):  # per-task selection mask over the frontier
            mask = np.ascontiguousarray(sel, dtype=np.uint8)
            if mask.shape != (opts.shard_end,):
                raise InvalidArgumentError("shard mask length must equal shard end (the frontier size)")
            opts.shard_mask = mask.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))
        else:
            opts.shard_stride = int(sel)
    if digest is not None:
        if not (isinstance(digest, np.ndarray) and digest.dtype == np.uint64 and digest.shape == (3,)
                and digest.flags.c_contiguous):
            raise InvalidArgumentError("digest must be a contiguous numpy uint64[3]")
        opts.digest = digest.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
        opts.digest_mod, opts.digest_rem = int(digest_sample[0]), int(digest_sample[1])
    if K_out is not None:
        check_device_matrix(K_out, n, "int64" if K_fixed else "float64", bra._t.ds.device_index)
    opts.count_screen_bytes = 1 if screen_bytes else 0   # measurement aid (bench roofline_screen)
    tie_buf, tie_count = None, ctypes.c_int64(0)
    if tie_log is not None:
        tie_buf = (_native.TieRecord * TIE_CAPACITY)()
        opts.tie_log = ctypes.cast(tie_buf, ctypes.POINTER(_native.TieRecord))
        opts.tie_capacity = TIE_CAPACITY
        opts.tie_count = ctypes.pointer(tie_count)
    log_count = ctypes.c_int64(0)
    cap = 0
    if quartet_log is not None and evaluate:
        ns = bra._t.ds.n_shells
        cap = int(min(ns ** 4, 1 << 22))
    while True:
        logbuf = None
        if cap:
            logbuf = np.empty((cap, 4), dtype=np.int32)
            opts.quartet_log = logbuf.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            opts.log_capacity = cap
            opts.log_count = ctypes.pointer(log_count)
        if K_out is None:
            K = np.empty((n, n))
            opts.K_on_device = 0
            kptr = K.ctypes.data_as(ctypes.c_void_p)
        else:
            K = K_out
            opts.K_on_device = 1
            kptr = ctypes.c_void_p(K_out.data_ptr())
        scale = ctypes.c_int(0)
        if K_fixed:
            if K_out is None or str(K_out.dtype) != "torch.int64":
                raise InvalidArgumentError("K_fixed needs K_out as a CUDA int64 tensor")
            opts.K_fixed = 1
            opts.K_scale = ctypes.pointer(scale)
        c = _native.Counters()
        _native.check(L.hxf_exchange(bra._t.handle, ket._t.handle, P._t.handle, ctypes.byref(opts),
                                     kptr, ctypes.byref(c), _native.current_stream()))
        if K_fixed:
            K = (K_out, int(scale.value))
        if cap and log_count.value > cap:
            cap = int(log_count.value)
            continue
        break
    if tie_log is not None:
        tie_log.extend(tie_buf[k].to_dict() for k in range(min(int(tie_count.value), TIE_CAPACITY)))
    log = None
    if cap:
        arr = logbuf[:log_count.value]
        order = np.lexsort((arr[:, 3], arr[:, 2], arr[:, 1], arr[:, 0]))
        log = [tuple(t) for t in arr[order].tolist()]
    return K, c, log


TIE_CAPACITY = 4096   # tie records returned per build (ties are rare; the counters hold the totals)


def last_timings():
    """Device stage times (ms) of the last build on this thread: [traversal, screen,
    eri stage, epilogue, total, eri kernels only, far-field classification + survivor sort]."""
    out = (ctypes.c_double * 7)()
    _native.lib().hxf_last_timings(out, 7)
    return list(out)


def _fill_common(dst, c):
    for k in ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
              "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
              "tasks_expanded", "children_spawned", "ties_task", "ties_leaf", "prim_quartets",
              "screen_bytes"):
        setattr(dst, k, int(getattr(c, k)))
    dst.culled_bound_ledger = float(c.culled_bound_ledger)


def build_exchange_naive(bra: ShellPairNode, ket: ShellPairNode, P: MatrixQuadtree,
                         tau_2e: float = 0.0, mode: str = "schwarz",
                         quartet_log: list | None = None, evaluate: bool = True,
                         threads: int = 1, tie_log: list | None = None):
    """K = -1/2 sum P_nl (mn|ls) by hextree traversal on the GPU.

    Returns (K, TraversalCounters).  Reference: exchange_naive.py:200-240.
    tie_log (extension): a list that receives the build's tie records (run_exchange).
    """
    K, c, log = run_exchange(bra, ket, P, tau_2e, mode, False, evaluate, quartet_log, tie_log=tie_log)
    out = TraversalCounters()
    _fill_common(out, c)
    if quartet_log is not None and log is not None:
        quartet_log.extend(log)
    return K, out


def build_exchange_symmetric(pairs: ShellPairNode, P: MatrixQuadtree, tau_2e: float = 0.0,
                             mode: str = "schwarz", quartet_log: list | None = None,
                             evaluate: bool = True, threads: int = 1, tie_log: list | None = None):
    """Canonical-pair (4-fold) exchange build on the GPU; K passes symmetrize_final.

    Returns (K, SymmetryCounters).  Reference: exchange_symmetry.py:364-409.
    tie_log (extension): a list that receives the build's tie records (run_exchange).
    """
    K, c, log = run_exchange(pairs, pairs, P, tau_2e, mode, True, evaluate, quartet_log,
                             symmetrize=evaluate, tie_log=tie_log)
    out = SymmetryCounters()
    _fill_common(out, c)
    out.links_culled_screening = int(c.links_culled_screening)
    out.links_culled_absent = int(c.links_culled_absent)
    for g, lab in enumerate(CASE_LABELS):
        out.case_tasks[lab] = int(c.case_tasks[g])
        out.case_leaf_tasks[lab] = int(c.case_leaf_tasks[g])
    if quartet_log is not None and log is not None:
        quartet_log.extend(log)
    return K, out


def build_exchange_eightfold(pairs: ShellPairNode, P: MatrixQuadtree, tau_2e: float = 0.0,
                             mode: str = "schwarz", quartet_log: list | None = None,
                             evaluate: bool = True, threads: int = 1):
    """(new) 8-fold mode: the 4-fold build folded bra <-> ket.

    Evaluates only canonical quartets with bra pair <= ket pair (product-tree
    tasks with bra node <= ket node; on a bra == ket leaf task, bra pair <= ket
    pair) and forms K = A + A^T, A = sum_{bra < ket} C(q) + 1/2 sum_{bra = ket} C(q),
    C(q) the 4-fold slot contributions of q: because P is symmetric, the
    mirror quartet's contributions are C(q)^T and its culling decisions equal
    q's.  The evaluated set is the 4-fold quartet_log folded to
    {unordered (bra pair, ket pair)}.  Counters count this traversal (about half
    the 4-fold tasks and quartets); K equals the 4-fold K within rounding.
    Returns (K, SymmetryCounters).
    """
    K, c, log = run_exchange(pairs, pairs, P, tau_2e, mode, "eightfold", evaluate, quartet_log)
    out = SymmetryCounters()
    _fill_common(out, c)
    out.links_culled_screening = int(c.links_culled_screening)
    out.links_culled_absent = int(c.links_culled_absent)
    for g, lab in enumerate(CASE_LABELS):
        out.case_tasks[lab] = int(c.case_tasks[g])
        out.case_leaf_tasks[lab] = int(c.case_leaf_tasks[g])
    if quartet_log is not None and log is not None:
        quartet_log.extend(log)
    return K, out


def dense_exchange_screened(pairs: ShellPairNode, P: MatrixQuadtree, tau_2e: float = 0.0,
                            mode: str = "schwarz", K_out=None, digest=None, sample=(1, 0)):
    """Direct-SCF twin on the GPU (oracle.py:69-108).

    Every ordered shell quartet (i,j,k,l) of live pairs with
    (f(Q_ij) |P|_jk) f(Q_kl) > tau_2e is evaluated -- no hierarchy -- by the
    same ERI stage into the same fixed-point K, so the result equals
    build_exchange_naive's K bit for bit when both evaluate the same set.
    sample = (m, r) evaluates only quartets whose first shell i has
    i % m == r (whole K rows of those shells' functions).  digest: optional
    numpy uint64[3] filled as in run_exchange.  Returns (K, TraversalCounters)
    with eri_shell_quartets and prim_quartets set; the reference's skipped
    bound sum is not formed (it cancels catastrophically at full size).
    """
    if not (tau_2e >= 0.0):
        raise InvalidArgumentError("tau_2e must be non-negative")
    if mode not in ("schwarz", "literal"):
        raise InvalidArgumentError(f"unknown screening mode {mode!r}")
    _check_same_partition(pairs, pairs, P)
    _require_root(pairs, "pairs")
    L = _native.lib()
    n = pairs.row.n_functions
    opts = _native.ExchangeOpts()
    opts.tau_2e = float(tau_2e)
    opts.mode = 0 if mode == "schwarz" else 1
    opts.evaluate = 1
    opts.digest_mod, opts.digest_rem = int(sample[0]), int(sample[1])
    if digest is not None:
        if not (isinstance(digest, np.ndarray) and digest.dtype == np.uint64 and digest.shape == (3,)):
            raise InvalidArgumentError("digest must be a contiguous numpy uint64[3]")
        opts.digest = digest.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64))
    if K_out is None:
        K = np.empty((n, n))
        opts.K_on_device = 0
        kptr = K.ctypes.data_as(ctypes.c_void_p)
    else:
        K = K_out
        opts.K_on_device = 1
        kptr = ctypes.c_void_p(K_out.data_ptr())
    c = _native.Counters()
    _native.check(L.hxf_exchange_direct(pairs._t.handle, P._t.handle, ctypes.byref(opts), kptr,
                                        ctypes.byref(c), _native.current_stream()))
    out = TraversalCounters()
    out.eri_shell_quartets = int(c.eri_shell_quartets)
    out.prim_quartets = int(c.prim_quartets)
    return K, out
