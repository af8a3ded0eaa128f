"""ctypes front end of oracle/direct_digest.c (TEST INFRASTRUCTURE ONLY).

The streamed direct-SCF rule (hexfock/oracle.py:69-108) reduced to an
order-independent digest of the evaluated quartet tuples, for full-size
parity at configs 4-5.  Only tests/ and bench.py's
CPU leg use this module.
"""
import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libdirect_digest.so")
_lib = None

MASK = (1 << 64) - 1


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            subprocess.run(["make", "-C", _HERE, "-s"], check=True)
        L = ctypes.CDLL(_LIB)
        L.direct_digest.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double,
                                    ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_int, ctypes.c_void_p]
        L.direct_digest.restype = ctypes.c_int
        _lib = L
    return _lib


def digest(q, pmax, tau, mode="schwarz", fourfold=False, sample=(1, 0), threads=None, eightfold=False):
    """(count, sum h, sum h(h)) of the direct-SCF evaluated set.

    q: (ns, ns) canonical Q (<= 0 where the pair is absent); pmax: (ns, ns)
    max |P| per shell block; fourfold: canonical tuples (the four-fold
    driver's quartet_log) instead of ordered ones; eightfold: the canonical
    tuples with (i,j) <= (k,l) (the fourfold set folded bra <-> ket).
    """
    q = np.ascontiguousarray(q, dtype=np.float64)
    pmax = np.ascontiguousarray(pmax, dtype=np.float64)
    ns = q.shape[0]
    assert q.shape == (ns, ns) and pmax.shape == (ns, ns)
    out = np.zeros(3, dtype=np.uint64)
    nt = threads or max(1, os.cpu_count() or 1)
    rc = _load().direct_digest(ns, q.ctypes.data, pmax.ctypes.data, float(tau),
                               0 if mode == "schwarz" else 1, 2 if eightfold else (1 if fourfold else 0),
                               int(sample[0]), int(sample[1]), nt, out.ctypes.data)
    if rc:
        raise MemoryError("direct_digest: allocation failed")
    return tuple(int(v) for v in out)


def _mix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def digest_of_tuples(tuples, ns, sample=(1, 0)):
    """The same digest of an explicit quartet list (e.g. a quartet_log)."""
    a = np.asarray(list(tuples), dtype=np.uint64).reshape(-1, 4)
    if sample[0] > 1:
        a = a[(a[:, 0] % np.uint64(sample[0])) == np.uint64(sample[1])]
    n = np.uint64(ns)
    with np.errstate(over="ignore"):
        key = ((a[:, 0] * n + a[:, 1]) * n + a[:, 2]) * n + a[:, 3]
        h = _mix64(key)
        h2 = _mix64(h)
    return (len(a), int(h.sum(dtype=np.uint64)) & MASK, int(h2.sum(dtype=np.uint64)) & MASK)
