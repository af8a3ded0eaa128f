"""Tie records (BASELINE north star: a bound within 1e-12 relative of its threshold
"must be logged"): thresholds set exactly on a bound the
device computes, at each of the three culling stages, and the record checked."""

import math

import numpy as np
import pytest

import paper_1401_6961_b200 as hx

pytestmark = pytest.mark.gpu


def _setup(leaf_size=4, tau_ovlp=1e-11, overlap_matrix=None):
    system = hx.generate_cluster(4, seed=11)
    system, _ = hx.hilbert_order(system)
    P = hx.build_density(system, hx.DensityModel())
    part = hx.build_partition(system, leaf_size=leaf_size)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=tau_ovlp, overlap_matrix=overlap_matrix)
    return system, P, part, pairs, hx.build_matrix_tree(P, part)


def test_no_ties_on_a_generic_threshold():
    _, _, _, pairs, Pt = _setup()
    ties = []
    _, c = hx.build_exchange_symmetric(pairs, Pt, 1e-8, tie_log=ties)
    assert ties == [] and c.ties_task == 0 and c.ties_leaf == 0
    assert pairs.overlap_ties == []


def test_leaf_tie_is_logged_with_its_quartet():
    system, P, _, pairs, Pt = _setup()
    log = []
    hx.build_exchange_naive(pairs, pairs, Pt, 1e-8, quartet_log=log)
    q = pairs._t.qmatrix()
    # the reference's leaf bound of a surviving quartet: (sqrt(Q_ij) |P_jk|) sqrt(Q_kl), s shells
    i, j, k, l = log[len(log) // 2]
    bound = (math.sqrt(q[i, j]) * abs(P[j, k])) * math.sqrt(q[k, l])
    assert bound > 1e-8
    ties = []
    _, c = hx.build_exchange_naive(pairs, pairs, Pt, bound, tie_log=ties)
    assert c.ties_leaf >= 1
    mine = [t for t in ties if t["stage"] == "leaf" and t["ids"] == (i, j, k, l)]
    assert len(mine) == 1
    t = mine[0]
    assert t["bound"] == bound and t["threshold"] == bound
    assert t["decision"] == "culled"          # keep iff bound > tau
    assert t["contribution"] == bound and t["slot"] == 0 and t["level"] == -1


def test_task_tie_is_logged_with_its_node():
    _, _, _, pairs, Pt = _setup()
    b = pairs.children[(0, 0)]
    p = Pt.children[(0, 0)]
    # exchange_naive.py:68-88: sorted factors, (lo * mid) * hi
    lo, mid, hi = sorted([math.sqrt(b.diag_norm), p.norm, math.sqrt(b.diag_norm)])
    bound = (lo * mid) * hi
    ties = []
    _, c = hx.build_exchange_naive(pairs, pairs, Pt, bound, tie_log=ties)
    assert c.ties_task >= 1
    mine = [t for t in ties if t["stage"] == "task" and t["level"] == 1 and t["ids"] == (0, 0, 0, 0)]
    assert len(mine) == 1
    assert mine[0]["bound"] == bound and mine[0]["decision"] == "culled"


def test_symmetric_task_tie_carries_the_slot():
    _, _, _, pairs, Pt = _setup()
    b = pairs.children[(0, 0)]
    k = pairs.children[(1, 1)]
    p = Pt.children[(0, 1)]      # slots g0..g3 of the task (0,0 | 1,1) all read P[0,1]
    lo, mid, hi = sorted([math.sqrt(b.diag_norm), p.norm, math.sqrt(k.diag_norm)])
    bound = (lo * mid) * hi
    ties = []
    _, c = hx.build_exchange_symmetric(pairs, Pt, bound, tie_log=ties)
    mine = [t for t in ties if t["stage"] == "task" and t["level"] == 1 and t["ids"] == (0, 0, 1, 1)]
    assert sorted(t["slot"] for t in mine) == [0, 1, 2, 3]
    assert c.ties_task >= 4


def test_overlap_tie_is_logged_at_build():
    system, _, part, _, _ = _setup()
    S = np.abs(hx.shell_overlap_matrix(system))
    leaves = part.leaves
    r, c = leaves[0], leaves[-1]
    tau = float(S[r.shell_lo:r.shell_hi, c.shell_lo:c.shell_hi].max())
    assert tau > 0.0
    pairs = hx.build_pair_tree(system, part, tau_ovlp=tau, overlap_matrix=S)
    ties = pairs.overlap_ties
    assert ties and all(t["stage"] == "overlap" and t["threshold"] == tau for t in ties)
    deepest = max(t["level"] for t in ties)
    hit = [t for t in ties if t["level"] == deepest and t["bound"] == tau]
    assert hit and all(t["decision"] == "kept" for t in hit)   # pruned iff max |S| < tau_ovlp
