"""Shared helpers for the test suite.

Markers: ``gpu`` tests need a B200 (run with ``-m gpu``); everything else runs
on CPU.  Golden fixtures under tests/golden were written by the reference
itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_1401_6961_b200.basis import BasisSystem, GaussianShell, assign_offsets  # noqa: E402

COUNTER_KEYS = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
                "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
                "tasks_expanded", "children_spawned")
SYM_KEYS = ("links_culled_screening", "links_culled_absent")
CASES = ("A", "B", "C", "D", "E", "F1", "F2", "H", "SPARSE")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def system_from_arrays(centers, prims, nprim, ls=None):
    shells = []
    off = 0
    for k in range(len(centers)):
        pr = [tuple(x) for x in prims[off:off + nprim[k]]]
        off += nprim[k]
        shells.append(GaussianShell(center=centers[k], primitives=pr,
                                    l=0 if ls is None else int(ls[k])))
    return BasisSystem(shells=assign_offsets(shells), atoms=[])


def counters_vec(c, sym):
    d = c.to_dict() if hasattr(c, "to_dict") else c
    v = [d[k] for k in COUNTER_KEYS]
    if sym:
        v += [d[k] for k in SYM_KEYS]
        v += [d["case_tasks"][k] for k in CASES] + [d["case_leaf_tasks"][k] for k in CASES]
    return np.asarray(v, dtype=np.int64)


def quartet_bits(log, n_sh):
    bits = np.zeros(n_sh ** 4, dtype=bool)
    if len(log):
        arr = np.asarray(log, dtype=np.int64).reshape(-1, 4)
        flat = ((arr[:, 0] * n_sh + arr[:, 1]) * n_sh + arr[:, 2]) * n_sh + arr[:, 3]
        assert len(np.unique(flat)) == len(flat), "duplicate quartets in log"
        bits[flat] = True
    return bits


def tree_walk(node, level=0, out=None):
    """Flatten a pair / matrix tree in sorted-child order (quadtree.py:398-404)."""
    out = [] if out is None else out
    norm = getattr(node, "norm", None)
    if norm is None:
        norm = node.diag_norm
    row, col = node.row, node.col
    rlo = getattr(row, "fn_lo", getattr(row, "flo", None))
    rhi = getattr(row, "fn_hi", getattr(row, "fhi", None))
    clo = getattr(col, "fn_lo", getattr(col, "flo", None))
    chi = getattr(col, "fn_hi", getattr(col, "fhi", None))
    out.append((level, rlo, rhi, clo, chi, norm, float(getattr(node, "pruned", False)),
                getattr(node, "rowsum_max", 0.0), getattr(node, "colsum_max", 0.0)))
    for key in sorted(getattr(node, "children", {}) or {}):
        tree_walk(node.children[key], level + 1, out)
    return out


def has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = load_golden(name)
        return cache[name]

    return get
