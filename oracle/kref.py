"""ctypes front end of oracle/kref.c (TEST INFRASTRUCTURE ONLY).

Independent CPU restatement for full-size parity:
the canonical Schwarz diagonal Q with overlap-pruned leaf blocks
(quadtree.py:284-337, integrals.py:58-64 / 219-222) and sampled rows of the
naive exchange K over the direct-SCF keep set (oracle.py:69-108), with C
Obara-Saika/HGP ERIs that share no code with the device kernels.  Shell
weights and the partition come from the Python oracle (hexfock_oracle.py),
not from the product package.  Only tests/ and bench.py's CPU leg use it.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import hexfock_oracle as ho

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libkref.so")
_lib = None
_P = ctypes.c_void_p


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            subprocess.run(["make", "-C", _HERE, "-s"], check=True)
        L = ctypes.CDLL(_LIB)
        L.kref_q.argtypes = [ctypes.c_int, _P, _P, _P, _P, _P, _P, ctypes.c_int, _P, _P,
                             ctypes.c_double, ctypes.c_int, _P]
        L.kref_q.restype = ctypes.c_int
        L.kref_rows.argtypes = [ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, _P, _P, _P, _P,
                                ctypes.c_double, ctypes.c_int, ctypes.c_int, _P, ctypes.c_int, _P,
                                ctypes.POINTER(ctypes.c_longlong)]
        L.kref_rows.restype = ctypes.c_int
        L.kref_eri_block.argtypes = [ctypes.c_int, _P, _P, _P, _P, _P, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _P]
        L.kref_eri_block.restype = ctypes.c_int
        _lib = L
    return _lib


class Basis:
    """Flat arrays of a system, normalised by the Python oracle."""

    def __init__(self, system):
        sh = ho.as_oracle_shells(system)
        self.shells = sh
        self.ns = len(sh)
        self.ctr = np.ascontiguousarray([s.center for s in sh], dtype=np.float64).reshape(-1, 3)
        self.l = np.asarray([s.l for s in sh], dtype=np.int32)
        self.nf = np.asarray([s.nfn for s in sh], dtype=np.int32)
        self.fn = np.asarray([s.fn for s in sh], dtype=np.int32)
        self.nfn = int(self.nf.sum())
        k = [len(s.exponents) for s in sh]
        self.poff = np.concatenate([[0], np.cumsum(k)]).astype(np.int32)
        self.ex = np.ascontiguousarray(np.concatenate([s.exponents for s in sh]), dtype=np.float64)
        self.w = np.ascontiguousarray(np.concatenate([s.weights for s in sh]), dtype=np.float64)
        self.sw = np.ascontiguousarray(np.concatenate([s.sweights for s in sh]), dtype=np.float64)

    def leaves(self, leaf_size):
        root = ho.build_partition(self.nf.tolist(), leaf_size)
        out, st = [], [root]
        while st:
            s = st.pop()
            if s.is_leaf:
                out.append((s.slo, s.shi))
            else:
                st.extend([s.right, s.left])
        out.sort()
        return np.asarray([a for a, _ in out], dtype=np.int32), np.asarray([b for _, b in out], dtype=np.int32)


def eri_block(basis, i, j, k, l):
    b = basis
    out = np.zeros(81)
    rc = _load().kref_eri_block(b.ns, b.ctr.ctypes.data, b.l.ctypes.data, b.poff.ctypes.data,
                                b.ex.ctypes.data, b.w.ctypes.data, i, j, k, l, out.ctypes.data)
    if rc:
        raise ValueError("kref: l > 1")
    n = [int(b.nf[x]) for x in (i, j, k, l)]
    return out[:n[0] * n[1] * n[2] * n[3]].reshape(n)


def q_matrix(basis, leaf_size, tau_ovlp, threads=None):
    """Dense canonical Q (ns x ns, symmetric); 0 for pairs in pruned leaf blocks."""
    b = basis
    lo, hi = b.leaves(leaf_size)
    q = np.empty((b.ns, b.ns))
    nt = threads or max(1, os.cpu_count() or 1)
    rc = _load().kref_q(b.ns, b.ctr.ctypes.data, b.l.ctypes.data, b.poff.ctypes.data, b.ex.ctypes.data,
                        b.w.ctypes.data, b.sw.ctypes.data, len(lo), lo.ctypes.data, hi.ctypes.data,
                        float(tau_ovlp), nt, q.ctypes.data)
    if rc:
        raise MemoryError("kref_q")
    return q


def pmax_blocks(basis, P):
    """max |P| over each shell-pair function block (ns x ns)."""
    A = np.abs(np.asarray(P, dtype=np.float64))
    if np.all(basis.nf == 1):
        return np.ascontiguousarray(A)
    starts = basis.fn.astype(np.intp)
    R = np.maximum.reduceat(A, starts, axis=0)
    return np.ascontiguousarray(np.maximum.reduceat(R, starts, axis=1))


def k_rows(basis, P, q, tau, rows, mode="schwarz", threads=None):
    """Rows of the naive K for shells `rows`: (function indices, K rows, #quartets)."""
    b = basis
    rows = np.ascontiguousarray(rows, dtype=np.int32)
    P = np.ascontiguousarray(P, dtype=np.float64)
    q = np.ascontiguousarray(q, dtype=np.float64)
    fidx = np.concatenate([b.fn[r] + np.arange(b.nf[r]) for r in rows]) if len(rows) else np.zeros(0, int)
    out = np.empty((len(fidx), b.nfn))
    nq = ctypes.c_longlong(0)
    nt = threads or max(1, os.cpu_count() or 1)
    rc = _load().kref_rows(b.ns, b.nfn, b.ctr.ctypes.data, b.l.ctypes.data, b.poff.ctypes.data,
                           b.ex.ctypes.data, b.w.ctypes.data, b.fn.ctypes.data, q.ctypes.data,
                           P.ctypes.data, float(tau), 0 if mode == "schwarz" else 1, len(rows),
                           rows.ctypes.data, nt, out.ctypes.data, ctypes.byref(nq))
    if rc:
        raise MemoryError("kref_rows")
    return fidx, out, int(nq.value)
