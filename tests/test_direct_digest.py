"""The streamed direct-SCF checker (oracle/direct_digest.c) against the Python
oracle's quartet logs (CPU).

Pins the C restatement used for full-size (configs 4-5) parity of the
evaluated quartet set: its naive digest must equal the
digest of the direct-SCF keep set (oracle.py:69-108) and of the hierarchical
naive driver's quartet_log (acceptance criterion 3); its four-fold digest must
equal the digest of the four-fold driver's canonical quartet_log.
"""

import numpy as np
import pytest

from oracle import direct_digest as dd
from oracle import hexfock_oracle as ho
from paper_1401_6961_b200 import configs

from conftest import load_golden, system_from_arrays


def _q_pm(shells, P):
    ns = len(shells)
    canon = ho.Pairs(shells, [(min(i, j), max(i, j)) for i in range(ns) for j in range(ns)])
    q = ho.diagonal_q(shells, canon).reshape(ns, ns)
    fn = np.asarray([sh.fn for sh in shells])
    nf = np.asarray([sh.nfn for sh in shells])
    return q, ho._pmax_block(P, fn, nf, fn, nf)


def _systems():
    g = load_golden("c1")
    c1 = system_from_arrays(g["centers"], g["prims"], g["nprim"])
    out = [("c1", c1, g["P"])]
    # a small p-shell water cluster (the c3-c5 recipe at 4 units)
    cfg = configs.cube_cluster(4, seed=7, name="w4")
    out.append(("w4", cfg.system, cfg.P))
    return out


@pytest.fixture(scope="module", params=[0, 1], ids=["c1", "w4"])
def case(request):
    name, system, P = _systems()[request.param]
    setup = ho.Setup(system, P, tau_ovlp=0.0, leaf_size=4 if name == "w4" else 10)
    q, pm = _q_pm(setup.shells, setup.P)
    return name, setup, q, pm


@pytest.mark.parametrize("tau,mode", [(1e-5, "schwarz"), (1e-3, "literal")])
def test_naive_digest_matches_direct_and_hierarchical_sets(case, tau, mode):
    _, setup, q, pm = case
    ns = q.shape[0]
    keep, _ = ho.screened_quartets(setup.shells, setup.P, tau, mode)
    direct = [tuple(t) for t in np.argwhere(keep)]
    want = dd.digest_of_tuples(direct, ns)
    assert dd.digest(q, pm, tau, mode) == want
    log = []
    setup.naive(tau, mode=mode, quartet_log=log)
    assert dd.digest_of_tuples(log, ns) == want        # criterion 3
    for sample in ((3, 1), (5, 0)):
        assert dd.digest(q, pm, tau, mode, sample=sample) == dd.digest_of_tuples(direct, ns, sample)


@pytest.mark.parametrize("tau,mode", [(1e-6, "schwarz"), (1e-3, "literal")])
def test_fourfold_digest_matches_symmetric_log(case, tau, mode):
    _, setup, q, pm = case
    ns = q.shape[0]
    log = []
    setup.symmetric(tau, mode=mode, quartet_log=log)
    assert dd.digest(q, pm, tau, mode, fourfold=True) == dd.digest_of_tuples(log, ns)
    assert dd.digest(q, pm, tau, mode, fourfold=True, sample=(4, 2)) == \
        dd.digest_of_tuples(log, ns, (4, 2))


def test_digest_is_thread_count_independent(case):
    _, _, q, pm = case
    a = dd.digest(q, pm, 1e-7, threads=1)
    b = dd.digest(q, pm, 1e-7, threads=5)
    assert a == b and a[0] > 0


def test_zero_tau_keeps_every_nonzero_bound(case):
    _, setup, q, pm = case
    fq = np.sqrt(np.maximum(q, 0.0))
    n = int(np.count_nonzero((fq[:, :, None, None] * pm[None, :, :, None]) * fq[None, None, :, :] > 0))
    assert dd.digest(q, pm, 0.0)[0] == n
