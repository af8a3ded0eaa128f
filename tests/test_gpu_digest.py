"""Full-size parity of the evaluated quartet set at the BASELINE configs
(SURVEY.md 8(c) item 2).

The device build returns an order-independent digest (count, sum h, sum h(h))
of its evaluated quartet tuples; the streamed CPU restatement of the
direct-SCF rule (oracle/direct_digest.c, pinned against the Python oracle in
tests/test_direct_digest.py) computes the same digest from the device's Q and
block-max |P| tables.  Equal digests = the hierarchical build evaluated exactly
the direct-SCF set (acceptance criterion 3) at c3/c4 in full and on a
deterministic 1/64 sample of first shells at c5.
"""

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


def _build(name):
    import torch
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs
    if name == "c5":
        cfg = configs.make(name, host_density=False)
        P = configs.decay_density_device(cfg.system, cfg.density_seed, "cuda")
    else:
        cfg = configs.make(name)
        P = torch.from_numpy(cfg.P).cuda()
    part = hx.build_partition(cfg.system, cfg.leaf_size)
    pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    Pt = hx.build_matrix_tree(P, part)
    return cfg, pairs, Pt, P


@pytest.fixture(scope="module", params=["c3", "c4", "c5"])
def built(request):
    return request.param, _build(request.param)


@pytest.mark.parametrize("sym", [False, True], ids=["naive", "fourfold"])
def test_evaluated_set_digest_matches_direct_scf(built, sym):
    import torch
    from oracle import direct_digest as dd
    from paper_1401_6961_b200 import exchange
    name, (cfg, pairs, Pt, P) = built
    sample = (64, 5) if name == "c5" else (1, 0)
    n = P.shape[0]
    K = torch.empty((n, n), dtype=torch.float64, device="cuda")
    dg = np.zeros(3, dtype=np.uint64)
    _, c, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, K_out=K,
                                    digest=dg, digest_sample=sample)
    del K
    torch.cuda.empty_cache()
    if sample[0] == 1:
        assert int(dg[0]) == c.eri_shell_quartets
    q = pairs._t.qmatrix()
    pm = Pt._t.pmax()
    want = dd.digest(q, pm, cfg.tau_2e, "schwarz", fourfold=sym, sample=sample)
    got = tuple(int(v) for v in dg)
    assert got == want, (name, sym, got, want)
