"""GPU direct-SCF twin and full-size K parity (8(c) item 2).

The twin (hxf_exchange_direct) evaluates the direct-SCF set (oracle.py:69-108)
without the hierarchy, through the same ERI stage and fixed-point K.
- small systems: twin K == the Python oracle's dense_exchange_screened K
  (<= 1e-10) and its evaluated set == the oracle's direct log (digest);
- c3 / c4 in full: twin K == hierarchical naive K bit for bit (the K
  accumulation is order-independent, so equal bits <=> equal evaluated sets
  and identical per-quartet arithmetic);
- c5: twin rows of a deterministic 1/64 sample of shells == the four-fold
  build's K rows (<= 1e-10 abs, the symmetrised K differs in rounding).
"""

import numpy as np
import pytest

from conftest import has_cuda, load_golden, system_from_arrays

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


def _small(name):
    from paper_1401_6961_b200 import configs
    if name == "c1":
        g = load_golden("c1")
        return system_from_arrays(g["centers"], g["prims"], g["nprim"]), g["P"], 10
    cfg = configs.cube_cluster(4, seed=7, name="w4")
    return cfg.system, cfg.P, 4


@pytest.mark.parametrize("name", ["c1", "w4"])
@pytest.mark.parametrize("tau", [1e-8, 1e-4])
def test_twin_matches_python_direct_scf(name, tau):
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import exchange
    from oracle import direct_digest as dd
    from oracle import hexfock_oracle as ho
    system, P, leaf = _small(name)
    part = hx.build_partition(system, leaf)
    pairs = hx.build_pair_tree(system, part, 0.0)
    Pt = hx.build_matrix_tree(P, part)
    dg = np.zeros(3, dtype=np.uint64)
    K, c = exchange.dense_exchange_screened(pairs, Pt, tau, digest=dg)
    shells = ho.as_oracle_shells(system)
    log = []
    K_ref, _ = ho.dense_exchange_screened(shells, np.asarray(P, float), tau, quartet_log=log)
    assert float(np.abs(K - K_ref).max()) <= 1e-10
    assert tuple(int(v) for v in dg) == dd.digest_of_tuples(log, len(shells))
    assert c.eri_shell_quartets == len(log)
    K_h, c_h = hx.build_exchange_naive(pairs, pairs, Pt, tau_2e=tau)
    assert np.array_equal(K, K_h)
    assert c.eri_shell_quartets == c_h.eri_shell_quartets


def _build(name):
    from test_gpu_digest import _build as b
    return b(name)


@pytest.mark.parametrize("name", ["c3", "c4"])
def test_twin_equals_hierarchical_naive_bitwise(name):
    import torch
    from paper_1401_6961_b200 import exchange
    cfg, pairs, Pt, P = _build(name)
    n = P.shape[0]
    K1 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    K2 = torch.empty_like(K1)
    _, c1, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", False, K_out=K1)
    _, c2 = exchange.dense_exchange_screened(pairs, Pt, cfg.tau_2e, K_out=K2)
    assert c1.eri_shell_quartets == c2.eri_shell_quartets
    assert c1.prim_quartets == c2.prim_quartets
    assert torch.equal(K1, K2)


def test_twin_sampled_rows_match_fourfold_c5():
    import torch
    from paper_1401_6961_b200 import exchange
    cfg, pairs, Pt, P = _build("c5")
    n = P.shape[0]
    K = torch.empty((n, n), dtype=torch.float64, device="cuda")
    exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", True, K_out=K)
    sample = (64, 5)
    fn = np.asarray([sh.function_offset for sh in cfg.system.shells])
    nf = np.asarray([sh.n_functions for sh in cfg.system.shells])
    rows = np.concatenate([np.arange(fn[i], fn[i] + nf[i])
                           for i in range(len(fn)) if i % sample[0] == sample[1]])
    rows_t = torch.from_numpy(rows).cuda()
    Kh = K[rows_t].clone()
    del K
    K2 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    _, c = exchange.dense_exchange_screened(pairs, Pt, cfg.tau_2e, K_out=K2, sample=sample)
    Kt = K2[rows_t]
    assert c.eri_shell_quartets > 0
    err = float((Kh - Kt).abs().max())
    scale = float(Kh.abs().max())
    assert err <= 1e-10, (err, scale)
