"""Partition and device-resident quadtrees behind the reference's tree API.

Mirror of ``hexfock/quadtree.py`` (reference paths below): the same function
names, signatures, attributes and exceptions, but the trees live on the B200.

  Span / Partition / build_partition ... quadtree.py:28-113 (host; ragged
                                         bisection, left tie-break)
  build_matrix_tree ................... quadtree.py:198-235 -> hxf_density_build
  build_pair_tree ..................... quadtree.py:284-337 -> hxf_pairs_build
  MatrixQuadtree / ShellPairNode ...... quadtree.py:116-142, 238-269 (lazy views
                                         of the device node arrays)
  transpose_view ...................... quadtree.py:154-195

The returned objects are lightweight views: node attributes are pulled from
the device the first time they are read (per level), so the reference's
call sequence  build_partition -> build_pair_tree -> build_matrix_tree ->
build_exchange_*  and its tree-inspecting tests work unchanged.
"""

from __future__ import annotations

import ctypes
import math
import weakref

import numpy as np

from . import _native
from .basis import BasisSystem, InvalidArgumentError

DEFAULT_LEAF_SIZE = 10


class Span:
    """Contiguous shell/function range; a node of the bisection tree."""

    __slots__ = ("shell_lo", "shell_hi", "fn_lo", "fn_hi", "left", "right", "__weakref__")

    def __init__(self, shell_lo, shell_hi, fn_lo, fn_hi, left=None, right=None):
        self.shell_lo, self.shell_hi = shell_lo, shell_hi
        self.fn_lo, self.fn_hi = fn_lo, fn_hi
        self.left, self.right = left, right

    @property
    def is_leaf(self) -> bool:
        return self.left is None

    @property
    def n_functions(self) -> int:
        return self.fn_hi - self.fn_lo

    def children(self):
        """Sub-spans for simultaneous descent; a leaf stands in for itself."""
        return (self,) if self.is_leaf else (self.left, self.right)

    def __repr__(self):
        return f"Span(shells {self.shell_lo}:{self.shell_hi}, fns {self.fn_lo}:{self.fn_hi})"


class Partition:
    def __init__(self, root: Span, leaf_size: int, system: BasisSystem | None = None):
        self.root = root
        self.leaf_size = leaf_size
        self.system = system
        self._levels = None
        self._device = None

    @property
    def levels(self):
        """Span lists per depth; ragged leaves repeat at deeper levels."""
        if self._levels is None:
            out = []
            frontier = [self.root]
            while True:
                out.append(frontier)
                if all(s.is_leaf for s in frontier):
                    break
                frontier = [c for s in frontier for c in s.children()]
            self._levels = out
        return [list(l) for l in self._levels]

    @property
    def leaves(self):
        out = []

        def walk(s):
            if s.is_leaf:
                out.append(s)
            else:
                walk(s.left)
                walk(s.right)

        walk(self.root)
        return out

    # -- device system (basis + level tables), created once per partition
    def device(self, device: int = 0):
        if self._device is None:
            if self.system is None:
                raise InvalidArgumentError("partition has no basis system attached")
            self._device = _DeviceSystem(self.system, self, device)
        return self._device


def build_partition(system: BasisSystem, leaf_size: int = DEFAULT_LEAF_SIZE) -> Partition:
    """Recursive bisection at the shell boundary nearest the function midpoint.

    Ties between equidistant boundaries break left; splitting stops once a
    span holds at most ``leaf_size`` functions (quadtree.py:90-113).
    """
    sizes = [int(sh.n_functions) for sh in system.shells]
    if leaf_size < max(sizes, default=1):
        raise InvalidArgumentError("leaf_size must be >= the largest shell")
    cum = np.concatenate([[0], np.cumsum(sizes)]).astype(int)

    def split(lo, hi):
        node = Span(lo, hi, int(cum[lo]), int(cum[hi]))
        if node.n_functions <= leaf_size:
            return node
        mid = (node.fn_lo + node.fn_hi) / 2.0
        cand = np.arange(lo + 1, hi)
        b = int(cand[int(np.argmin(np.abs(cum[cand] - mid)))])
        node.left = split(lo, b)
        node.right = split(b, hi)
        return node

    return Partition(root=split(0, len(sizes)), leaf_size=leaf_size, system=system)


def _s_proxy_weights(sh) -> np.ndarray:
    """s-normalised weights of a shell's primitives (overlap pruning proxy)."""
    if int(getattr(sh, "l", 0)) == 0:
        return np.asarray(sh.weights, dtype=float)
    exps = np.asarray([e for e, _ in sh.primitives], dtype=float)
    coefs = np.asarray([c for _, c in sh.primitives], dtype=float)
    w = coefs * (2.0 * exps / np.pi) ** 0.75
    p = exps[:, None] + exps[None, :]
    s = np.sum(w[:, None] * w[None, :] * (np.pi / p) ** 1.5)
    return w / math.sqrt(s)


class _DeviceSystem:
    """Owns the hxf_system handle: basis arrays + partition level tables."""

    def __init__(self, system, partition, device=0):
        L = _native.lib()
        shells = system.shells
        ns = len(shells)
        centers = np.ascontiguousarray([sh.center for sh in shells], dtype=np.float64).reshape(ns, 3)
        lval = np.asarray([int(getattr(sh, "l", 0)) for sh in shells], dtype=np.int32)
        nfn = np.asarray([int(sh.n_functions) for sh in shells])
        if np.any(nfn != np.where(lval == 0, 1, 3)):
            raise InvalidArgumentError("shell n_functions must be 1 (s) or 3 (p)")
        nprim = [len(sh.exponents) for sh in shells]
        prim_off = np.concatenate([[0], np.cumsum(nprim)]).astype(np.int32)
        exps = np.ascontiguousarray(np.concatenate([sh.exponents for sh in shells]), dtype=np.float64)
        w = np.ascontiguousarray(np.concatenate([sh.weights for sh in shells]), dtype=np.float64)
        sw = np.ascontiguousarray(np.concatenate([_s_proxy_weights(sh) for sh in shells]),
                                  dtype=np.float64)
        levels = partition.levels
        self.levels = levels
        self.index = [{id(s): k for k, s in enumerate(lvl)} for lvl in levels]
        off = np.concatenate([[0], np.cumsum([len(l) for l in levels])]).astype(np.int32)
        cols = {k: [] for k in ("slo", "shi", "flo", "fhi", "k0", "k1")}
        for L_, lvl in enumerate(levels):
            nxt = self.index[L_ + 1] if L_ + 1 < len(levels) else None
            for s in lvl:
                cols["slo"].append(s.shell_lo)
                cols["shi"].append(s.shell_hi)
                cols["flo"].append(s.fn_lo)
                cols["fhi"].append(s.fn_hi)
                if nxt is None:
                    cols["k0"].append(-1)
                    cols["k1"].append(-1)
                elif s.is_leaf:
                    cols["k0"].append(nxt[id(s)])
                    cols["k1"].append(-1)
                else:
                    cols["k0"].append(nxt[id(s.left)])
                    cols["k1"].append(nxt[id(s.right)])
        arr = {k: np.asarray(v, dtype=np.int32) for k, v in cols.items()}
        h = ctypes.c_void_p()
        _native.check(L.hxf_system_create(
            int(device), ns, _native.ptr(centers), _native.ptr(lval), _native.ptr(prim_off),
            _native.ptr(exps), _native.ptr(w), _native.ptr(sw), len(levels), _native.ptr(off),
            _native.ptr(arr["slo"]), _native.ptr(arr["shi"]), _native.ptr(arr["flo"]),
            _native.ptr(arr["fhi"]), _native.ptr(arr["k0"]), _native.ptr(arr["k1"]),
            ctypes.byref(h)))
        self.handle = h
        self.device_index = int(device)
        self.n_shells = ns
        self.n_functions = int(nfn.sum())
        self.shell_fn = np.concatenate([[0], np.cumsum(nfn)]).astype(np.int64)
        weakref.finalize(self, L.hxf_system_destroy, h)


# ----------------------------------------------------------------- density tree

class _DensityTree:
    def __init__(self, partition, dense, zero_drop, device_P=None):
        ds = partition.device()
        self.partition = partition
        self.ds = ds
        self.host_dense = dense
        h = ctypes.c_void_p()
        if device_P is not None:
            _native.check(_native.lib().hxf_density_build(ds.handle, _native.ptr(device_P), 1,
                                                          float(zero_drop), _native.current_stream(),
                                                          ctypes.byref(h)))
        else:
            _native.check(_native.lib().hxf_density_build(ds.handle, _native.ptr(dense), 0,
                                                          float(zero_drop), _native.current_stream(),
                                                          ctypes.byref(h)))
        self.handle = h
        weakref.finalize(self, _native.lib().hxf_density_destroy, h)
        self._norms = {}
        # weak cache: views reference their tree, so a strong cache would make a
        # cycle and defer freeing the device arrays to the cyclic GC
        self._views = weakref.WeakValueDictionary()

    def norms(self, level):
        v = self._norms.get(level)
        if v is None:
            n = len(self.ds.levels[level])
            v = np.empty(n * n)
            _native.check(_native.lib().hxf_density_download(self.handle, level, _native.ptr(v)))
            self._norms[level] = v
        return v

    def pmax(self):
        """max |P| over each shell block (n_shells x n_shells)."""
        ns = self.ds.n_shells
        v = np.empty(ns * ns)
        _native.check(_native.lib().hxf_density_download_pmax(self.handle, _native.ptr(v)))
        return v.reshape(ns, ns)

    def view(self, level, r, c):
        key = (level, r, c)
        v = self._views.get(key)
        if v is None:
            v = MatrixQuadtree(self, level, r, c)
            self._views[key] = v
        return v


class MatrixQuadtree:
    """View of one density-quadtree node (quadtree.py:116-142)."""

    __slots__ = ("_t", "_level", "_r", "_c", "row", "col", "__weakref__")

    def __init__(self, tree, level, r, c):
        self._t, self._level, self._r, self._c = tree, level, r, c
        lv = tree.ds.levels[level]
        self.row, self.col = lv[r], lv[c]

    @property
    def norm(self) -> float:
        n = len(self._t.ds.levels[self._level])
        v = float(self._t.norms(self._level)[self._r * n + self._c])
        return max(v, 0.0)

    @property
    def is_leaf(self) -> bool:
        return self.row.is_leaf and self.col.is_leaf

    @property
    def leaf(self):
        if not self.is_leaf:
            return None
        return self._t.host_dense[self.row.fn_lo:self.row.fn_hi, self.col.fn_lo:self.col.fn_hi]

    def _present(self, level, r, c) -> bool:
        n = len(self._t.ds.levels[level])
        return self._t.norms(level)[r * n + c] >= 0.0

    @property
    def children(self):
        if self.is_leaf:
            return {}
        L = self._level
        nxt = self._t.ds.index[L + 1]
        out = {}
        for a, rs in enumerate(self.row.children()):
            for b, cs in enumerate(self.col.children()):
                r2, c2 = nxt[id(rs)], nxt[id(cs)]
                if self._present(L + 1, r2, c2):
                    out[(a, b)] = self._t.view(L + 1, r2, c2)
        return out

    def child(self, a, b):
        if self.is_leaf:
            return self if (a, b) == (0, 0) else None
        return self.children.get((a, b))

    def dense(self) -> np.ndarray:
        out = np.zeros((self.row.n_functions, self.col.n_functions))
        self._fill(out, self.row.fn_lo, self.col.fn_lo)
        return out

    def _fill(self, out, r0, c0):
        if self.is_leaf:
            out[self.row.fn_lo - r0:self.row.fn_hi - r0, self.col.fn_lo - c0:self.col.fn_hi - c0] = self.leaf
            return
        for ch in self.children.values():
            ch._fill(out, r0, c0)


class TransposedQuadtree:
    """Constant-cost logical transpose of a MatrixQuadtree node."""

    __slots__ = ("base",)

    def __init__(self, base):
        self.base = base

    row = property(lambda self: self.base.col)
    col = property(lambda self: self.base.row)
    norm = property(lambda self: self.base.norm)
    is_leaf = property(lambda self: self.base.is_leaf)

    @property
    def leaf(self):
        lf = self.base.leaf
        return None if lf is None else lf.T

    def child(self, a, b):
        ch = self.base.child(b, a)
        return None if ch is None else TransposedQuadtree(ch)

    def dense(self):
        return self.base.dense().T


def transpose_view(node):
    """Logical transpose; applying it twice returns the original node."""
    if isinstance(node, TransposedQuadtree):
        return node.base
    return TransposedQuadtree(node)


def build_matrix_tree(dense, partition: Partition, zero_drop: float = 0.0) -> MatrixQuadtree:
    """Density quadtree on the device (quadtree.py:198-235).

    ``dense`` is a host array (reference API) or a CUDA tensor (device input,
    no host copy).  Leaves whose block is exactly zero, or whose norm is
    <= zero_drop, are absent; interior norms are correctly rounded RSS of the
    present children.
    """
    n = partition.root.n_functions
    if hasattr(dense, "is_cuda") and dense.is_cuda:
        if tuple(dense.shape) != (n, n):
            raise InvalidArgumentError(f"matrix shape {tuple(dense.shape)} does not match partition size {n}")
        t = _DensityTree(partition, None, zero_drop, device_P=dense.contiguous())
        return t.view(0, 0, 0)
    dense = np.ascontiguousarray(np.asarray(dense, dtype=float))
    if dense.shape != (n, n):
        raise InvalidArgumentError(f"matrix shape {dense.shape} does not match partition size {n}")
    t = _DensityTree(partition, dense, zero_drop)
    return t.view(0, 0, 0)


# ----------------------------------------------------------------- pair tree

class _PairTree:
    def __init__(self, partition, tau_ovlp, s_abs=None):
        ds = partition.device()
        self.partition = partition
        self.ds = ds
        self.tau_ovlp = tau_ovlp
        h = ctypes.c_void_p()
        if s_abs is None:
            _native.check(_native.lib().hxf_pairs_build(ds.handle, float(tau_ovlp),
                                                        _native.current_stream(), ctypes.byref(h)))
        else:
            on_dev = 1 if (hasattr(s_abs, "is_cuda") and s_abs.is_cuda) else 0
            _native.check(_native.lib().hxf_pairs_build_ovlp(ds.handle, float(tau_ovlp), _native.ptr(s_abs),
                                                             on_dev, _native.current_stream(),
                                                             ctypes.byref(h)))
        self.handle = h
        weakref.finalize(self, _native.lib().hxf_pairs_destroy, h)
        self._lvl = {}
        self._q = None
        # weak cache: views reference their tree, so a strong cache would make a
        # cycle and defer freeing the device arrays to the cyclic GC
        self._views = weakref.WeakValueDictionary()

    def level(self, L):
        v = self._lvl.get(L)
        if v is None:
            n = len(self.ds.levels[L])
            norm, rs, cs = np.empty(n * n), np.empty(n * n), np.empty(n * n)
            pr = np.empty(n * n, dtype=np.uint8)
            _native.check(_native.lib().hxf_pairs_download(self.handle, L, _native.ptr(norm),
                                                           _native.ptr(rs), _native.ptr(cs),
                                                           _native.ptr(pr)))
            v = (norm, rs, cs, pr.astype(bool))
            self._lvl[L] = v
        return v

    def overlap_ties(self):
        """Overlap-pruning comparisons (block max |S| < tau_ovlp, quadtree.py:296-299)
        within 1e-12 relative of tau_ovlp, found when the tree was built: a list of
        tie-record dicts (stage "overlap", level, level-local span ids, |S|, tau_ovlp)."""
        n = ctypes.c_int64(0)
        _native.check(_native.lib().hxf_pairs_ties(self.handle, None, 0, ctypes.byref(n)))
        k = min(int(n.value), 4096)
        if not k:
            return []
        buf = (_native.TieRecord * k)()
        _native.check(_native.lib().hxf_pairs_ties(self.handle, ctypes.cast(buf, ctypes.POINTER(_native.TieRecord)),
                                                   k, ctypes.byref(n)))
        return [buf[i].to_dict() for i in range(k)]

    def qmatrix(self):
        if self._q is None:
            ns = self.ds.n_shells
            q = np.empty(ns * ns)
            _native.check(_native.lib().hxf_pairs_download_q(self.handle, _native.ptr(q)))
            self._q = q.reshape(ns, ns)
        return self._q

    def view(self, L, r, c):
        key = (L, r, c)
        v = self._views.get(key)
        if v is None:
            v = ShellPairNode(self, L, r, c)
            self._views[key] = v
        return v


class ShellPairNode:
    """View of one shell-pair quadtree node (quadtree.py:238-269)."""

    __slots__ = ("_t", "_level", "_r", "_c", "row", "col", "__weakref__")

    def __init__(self, tree, level, r, c):
        self._t, self._level, self._r, self._c = tree, level, r, c
        lv = tree.ds.levels[level]
        self.row, self.col = lv[r], lv[c]

    def _get(self, k):
        n = len(self._t.ds.levels[self._level])
        return self._t.level(self._level)[k][self._r * n + self._c]

    @property
    def pruned(self) -> bool:
        return bool(self._get(3))

    @property
    def diag_norm(self) -> float:
        return float(self._get(0))

    @property
    def rowsum_max(self) -> float:
        return float(self._get(1))

    @property
    def colsum_max(self) -> float:
        return float(self._get(2))

    @property
    def overlap_ties(self):
        """(extension) tie records of the tree's overlap pruning."""
        return self._t.overlap_ties()

    @property
    def is_leaf(self) -> bool:
        return self.row.is_leaf and self.col.is_leaf

    @property
    def diag(self):
        """(ab|ab) block in canonical orientation (leaf nodes only)."""
        if not self.is_leaf or self.pruned:
            return None
        q = self._t.qmatrix()
        return q[self.row.shell_lo:self.row.shell_hi, self.col.shell_lo:self.col.shell_hi].copy()

    @property
    def children(self):
        if self.is_leaf or self.pruned:
            return {}
        L = self._level
        nxt = self._t.ds.index[L + 1]
        out = {}
        for a, rs in enumerate(self.row.children()):
            for b, cs in enumerate(self.col.children()):
                out[(a, b)] = self._t.view(L + 1, nxt[id(rs)], nxt[id(cs)])
        return out

    def child(self, a, b):
        if self.is_leaf:
            return self if (a, b) == (0, 0) else None
        return self.children.get((a, b))


def build_pair_tree(system: BasisSystem, partition: Partition, tau_ovlp: float = 0.0,
                    overlap_matrix=None) -> ShellPairNode:
    """Shell-pair quadtree with overlap pruning, built on the device.

    A node is pruned iff every shell-pair overlap magnitude in its span is
    below tau_ovlp (quadtree.py:284-337).  ``overlap_matrix`` (n_shells x
    n_shells, host array or CUDA tensor) replaces the computed overlaps for the
    pruning decisions, as in the reference (|S| of the given matrix, block max
    per node, not assumed symmetric); Q and the ERIs are unaffected.
    """
    s_abs = None
    if overlap_matrix is not None:
        ns = len(system.shells)
        if hasattr(overlap_matrix, "is_cuda") and overlap_matrix.is_cuda:
            import torch
            s_abs = overlap_matrix.detach().to(torch.float64).abs().contiguous()
        else:
            s_abs = np.ascontiguousarray(np.abs(np.asarray(overlap_matrix, dtype=float)))
        if tuple(s_abs.shape) != (ns, ns):
            raise InvalidArgumentError(f"overlap_matrix must be ({ns}, {ns}), got {tuple(s_abs.shape)}")
    if partition.system is None:
        partition.system = system
    elif partition.system is not system:
        if len(partition.system.shells) != len(system.shells):
            raise InvalidArgumentError("system does not match the partition")
    t = _PairTree(partition, tau_ovlp, s_abs)
    return t.view(0, 0, 0)


def shell_overlap_matrix(system: BasisSystem) -> np.ndarray:
    """Exactly symmetric contracted (s-proxy) overlap matrix -- host utility.

    API mirror of quadtree.py:272-281 for callers and tests; the device path
    computes block maxima itself and never calls this.
    """
    shells = system.shells
    n = len(shells)
    sw = [_s_proxy_weights(sh) for sh in shells]
    s = np.zeros((n, n))
    for i in range(n):
        for j in range(i, n):
            a, b = shells[i], shells[j]
            d = a.center - b.center
            r2 = float(np.dot(d, d))
            ea, eb = a.exponents[:, None], b.exponents[None, :]
            p = ea + eb
            v = float(np.sum(sw[i][:, None] * sw[j][None, :] * (np.pi / p) ** 1.5 *
                             np.exp(-ea * eb / p * r2)))
            s[i, j] = v
            s[j, i] = v
    return s
