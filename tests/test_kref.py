"""Pin the independent C restatement (oracle/kref.c) against the Python oracle.

kref is what the full-size GPU parity tests compare K rows and the Schwarz
diagonal against (tests/test_gpu_full_parity.py), so it is itself checked
here on CPU against oracle/hexfock_oracle.py, whose s path is pinned to
reference-written goldens and whose p path is pinned by the derivative
identity (tests/test_oracle_pshell.py):
  - every contracted block class (ss|ss) ... (pp|pp) to 1e-13 relative;
  - Q with overlap-pruned leaf blocks equal to the oracle's pair tree;
  - K rows equal to dense_exchange_screened (the direct-SCF oracle) to 1e-13.
"""

import itertools

import numpy as np
import pytest

from oracle import hexfock_oracle as ho
from oracle import kref
from paper_1401_6961_b200 import configs


def _sys(name, units=None):
    kw = {} if units is None else {"n_units": units}
    return configs.make(name, **kw)


@pytest.fixture(scope="module")
def small_p():
    return _sys("c3", units=6)


def test_eri_blocks_match_python_oracle(small_p):
    cfg = small_p
    b = kref.Basis(cfg.system)
    sh = b.shells
    rng = np.random.default_rng(7)
    by_l = [np.nonzero(b.l == v)[0] for v in (0, 1)]
    for cls in itertools.product((0, 1), repeat=4):
        for _ in range(6):
            q = [int(rng.choice(by_l[v])) for v in cls]
            bra = ho.Pairs(sh, [(q[0], q[1])])
            ket = ho.Pairs(sh, [(q[2], q[3])])
            want = ho.eri_blocks(sh, bra, ket, [0], [0])[0]
            got = kref.eri_block(b, *q)
            scale = max(np.abs(want).max(), 1e-300)
            assert np.abs(got - want).max() <= 1e-13 * scale, (q, cls)


@pytest.mark.parametrize("tau_ovlp", [0.0, 1e-11, 1e-4])
def test_q_matrix_matches_oracle_pair_tree(small_p, tau_ovlp):
    cfg = small_p
    b = kref.Basis(cfg.system)
    q = kref.q_matrix(b, cfg.leaf_size, tau_ovlp, threads=2)
    ns = b.ns
    canon = ho.Pairs(b.shells, [(min(i, j), max(i, j)) for i in range(ns) for j in range(ns)])
    qo = ho.diagonal_q(b.shells, canon).reshape(ns, ns)
    st = ho.Setup(cfg.system, cfg.P, tau_ovlp=tau_ovlp, leaf_size=cfg.leaf_size)
    present = np.zeros((ns, ns), dtype=bool)

    def walk(node):
        if node.pruned:
            return
        if node.is_leaf:
            present[node.row.slo:node.row.shi, node.col.slo:node.col.shi] = True
            return
        for c in node.children.values():
            walk(c)

    walk(st.pairs)
    assert np.array_equal(q > 0, present)
    np.testing.assert_allclose(q[present], qo[present], rtol=1e-13, atol=0)


@pytest.mark.parametrize("name,units", [("c1", None), ("c3", 5)])
def test_k_rows_match_direct_scf_oracle(name, units):
    cfg = _sys(name, units)
    b = kref.Basis(cfg.system)
    q = kref.q_matrix(b, cfg.leaf_size, 0.0, threads=2)
    K_ref, _ = ho.dense_exchange_screened(b.shells, cfg.P, cfg.tau_2e)
    rows = np.arange(b.ns)
    fidx, Kr, nq = kref.k_rows(b, cfg.P, q, cfg.tau_2e, rows, threads=2)
    keep, _ = ho.screened_quartets(b.shells, cfg.P, cfg.tau_2e)
    assert nq == int(keep.sum())
    assert np.abs(Kr - K_ref[fidx]).max() <= 1e-13


def test_pmax_blocks(small_p):
    cfg = small_p
    b = kref.Basis(cfg.system)
    pm = kref.pmax_blocks(b, cfg.P)
    want = ho._pmax_block(cfg.P, b.fn, b.nf, b.fn, b.nf)
    assert np.array_equal(pm, want)
