"""Device input preparation: Hilbert reordering and the
partition build on the GPU.

``hilbert_order_device`` is the drop-in for the reference's host pre-pass
``hilbert_order`` (basis.py:309-331, keys from ``hilbert_index_3d``,
basis.py:275-306): same arguments, same (system, permutation) result, same
InvalidArgumentError for ``bits_per_axis`` outside [1, 20] — computed by
``hxf_hilbert_order`` (csrc/prep.cu): lattice + Skilling keys per shell in one
kernel, a stable cub radix sort for the permutation.  Bitwise the host result
(tests/test_gpu_prep.py).  No CPU fallback: without a device it raises.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .basis import BasisSystem, GaussianShell, InvalidArgumentError, assign_offsets
from .quadtree import DEFAULT_LEAF_SIZE, Partition, Span


def hilbert_keys_and_perm(centers, bits_per_axis: int = 10):
    """(sorted keys uint64, stable permutation int64) of an (n, 3) float64 array of
    shell centres; host buffers in and out (hxf_hilbert_order, on_device=0)."""
    c = np.ascontiguousarray(np.asarray(centers, dtype=np.float64).reshape(-1, 3))
    n = c.shape[0]
    perm = np.empty(n, dtype=np.int64)
    keys = np.empty(n, dtype=np.uint64)
    _native.check(_native.lib().hxf_hilbert_order(
        _native.ptr(c), ctypes.c_int64(n), ctypes.c_int(int(bits_per_axis)), ctypes.c_int(0),
        _native.ptr(perm), _native.ptr(keys), _native.current_stream()))
    return keys, perm


def hilbert_order_device(system: BasisSystem, bits_per_axis: int = 10):
    """Stable Hilbert sort of shells on the GPU; returns (system, shell permutation)
    exactly like ``basis.hilbert_order`` (basis.py:309-331)."""
    if not 1 <= bits_per_axis <= 20:
        raise InvalidArgumentError("bits_per_axis must be in [1, 20]")
    centers = np.array([sh.center for sh in system.shells], dtype=np.float64)
    _, perm = hilbert_keys_and_perm(centers, bits_per_axis)
    shells = [GaussianShell(center=system.shells[k].center.copy(),
                            primitives=list(system.shells[k].primitives),
                            l=int(getattr(system.shells[k], "l", 0)))
              for k in perm]
    return BasisSystem(shells=assign_offsets(shells), atoms=system.atoms), perm


def partition_levels_device(shell_nfunc, leaf_size: int = DEFAULT_LEAF_SIZE):
    """Level tables of the bisection (hxf_partition_build, csrc/prep.cu): a list per
    level of (shell_lo, shell_hi) int32 arrays, leaves repeating as in
    Partition.levels (quadtree.py:90-113)."""
    sizes = np.ascontiguousarray(np.asarray(shell_nfunc, dtype=np.int32).reshape(-1))
    n = sizes.size
    L = _native.lib()
    cap_spans, cap_levels = max(16, 4 * (n + 1)), 64
    for _ in range(2):
        lo = np.empty(cap_spans, dtype=np.int32)
        hi = np.empty(cap_spans, dtype=np.int32)
        off = np.empty(cap_levels, dtype=np.int64)
        n_spans, n_levels = ctypes.c_int64(0), ctypes.c_int(0)
        rc = L.hxf_partition_build(_native.ptr(sizes), ctypes.c_int64(n), ctypes.c_int(int(leaf_size)),
                                   _native.ptr(lo), _native.ptr(hi), ctypes.c_int64(cap_spans),
                                   _native.ptr(off), ctypes.c_int(cap_levels),
                                   ctypes.byref(n_spans), ctypes.byref(n_levels),
                                   _native.current_stream())
        if rc == _native.HXF_EINVAL and n_spans.value > 0 and (
                n_spans.value > cap_spans or n_levels.value + 1 > cap_levels):
            cap_spans, cap_levels = int(n_spans.value), int(n_levels.value) + 1
            continue
        _native.check(rc)
        return [(lo[off[k]:off[k + 1]].copy(), hi[off[k]:off[k + 1]].copy())
                for k in range(n_levels.value)]
    raise RuntimeError("hxf_partition_build: capacity retry failed")  # pragma: no cover


def build_partition_device(system: BasisSystem, leaf_size: int = DEFAULT_LEAF_SIZE) -> Partition:
    """Drop-in for ``quadtree.build_partition`` with the bisection computed on the GPU:
    the same Span tree (shell and function bounds, children) as the host rules."""
    sizes = [int(sh.n_functions) for sh in system.shells]
    levels = partition_levels_device(sizes, leaf_size)
    cum = np.concatenate([[0], np.cumsum(sizes)]).astype(int)

    def span(a, b):
        return Span(int(a), int(b), int(cum[a]), int(cum[b]))

    split = {}
    for (lo, hi), (nlo, nhi) in zip(levels[:-1], levels[1:]):
        j = 0
        for a, z in zip(lo.tolist(), hi.tolist()):
            if nlo[j] == a and nhi[j] == z:   # a leaf repeats at the next level
                j += 1
            else:                             # children (a, b), (b, z)
                split[(a, z)] = int(nhi[j])
                j += 2

    def grow(a, z):
        node = span(a, z)
        b = split.get((a, z))
        if b is not None:
            node.left, node.right = grow(a, b), grow(b, z)
        return node

    return Partition(root=grow(int(levels[0][0][0]), int(levels[0][1][0])), leaf_size=leaf_size,
                     system=system)
