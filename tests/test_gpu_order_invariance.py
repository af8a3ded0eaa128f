"""The work-order changes of round 2 leave the result alone.

* Leaf tasks in bra-node-major order, the leaf screen's task-run length and grid, and the
  binning's column count only reorder work: the counters and the evaluated-set digest are
  identical and K -- accumulated with integer atomics in fixed point -- is bitwise the same.
* The far-field collapse (a same-centre (ss| pair enters the far-field ERI kernels as one
  point charge) changes the arithmetic of those quartets only by rounding: identical
  counters and set, K within 1e-13, fewer primitive quartets.
"""

import os

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_cuda(), reason="needs CUDA")]


class _env:
    def __init__(self, **kv):
        self.kv = kv

    def __enter__(self):
        self.old = {k: os.environ.get(k) for k in self.kv}
        os.environ.update({k: str(v) for k, v in self.kv.items()})

    def __exit__(self, *a):
        for k, v in self.old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _cdict(c):
    """The raw hxf_counters struct as a dict (arrays as lists)."""
    out = {}
    for name, _ in c._fields_:
        v = getattr(c, name)
        out[name] = list(v) if hasattr(v, "__len__") else v
    return out


def _setup(units=96):
    import torch
    import paper_1401_6961_b200 as hx
    from paper_1401_6961_b200 import configs
    cfg = configs.cube_cluster(units, 21, "c3")
    part = hx.build_partition(cfg.system, cfg.leaf_size)
    P = torch.from_numpy(cfg.P).cuda()
    return hx, cfg, part, P


def _run(hx, cfg, part, P, pairs, sym):
    import torch
    from paper_1401_6961_b200 import exchange
    n = P.shape[0]
    Pt = hx.build_matrix_tree(P, part)
    K = torch.empty((n, n), dtype=torch.float64, device="cuda")
    dg = np.zeros(3, dtype=np.uint64)
    _, c, _ = exchange.run_exchange(pairs, pairs, Pt, cfg.tau_2e, "schwarz", sym, K_out=K, digest=dg)
    return K, c, dg


@pytest.mark.parametrize("sym", [False, True, "eightfold"], ids=["naive", "fourfold", "eightfold"])
def test_work_order_does_not_change_K(sym):
    import torch
    hx, cfg, part, P = _setup()
    pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    K0, c0, d0 = _run(hx, cfg, part, P, pairs, sym)
    assert c0.eri_shell_quartets > 10 ** 6
    for env in ({"HXF_LEAF_SORT": 0}, {"HXF_LEAF_SORT": 0, "HXF_TASK_BLOCK": 1}, {"HXF_TASK_BLOCK": 5},
                {"HXF_SCREEN_BLOCKS": 3, "HXF_TASK_BLOCK": 64}, {"HXF_BIN_BLOCKS": 1},
                {"HXF_BIN_BLOCKS": 64, "HXF_SCREEN_BLOCKS": 12}):
        with _env(**env):
            K1, c1, d1 = _run(hx, cfg, part, P, pairs, sym)
        assert torch.equal(K0, K1), env
        assert np.array_equal(d0, d1), env
        a, b = _cdict(c0), _cdict(c1)
        led0, led1 = a.pop("culled_bound_ledger"), b.pop("culled_bound_ledger")
        assert a == b, env
        assert led1 == pytest.approx(led0, rel=1e-13), env
        assert c0.prim_quartets == c1.prim_quartets, env


def test_far_field_collapse_is_a_rounding_level_change():
    import torch
    hx, cfg, part, P = _setup(128)
    pairs = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    with _env(HXF_FAR_COLLAPSE=0):
        pairs_full = hx.build_pair_tree(cfg.system, part, cfg.tau_ovlp)
    for sym in (False, True):
        K1, c1, d1 = _run(hx, cfg, part, P, pairs, sym)
        K0, c0, d0 = _run(hx, cfg, part, P, pairs_full, sym)
        assert np.array_equal(d0, d1)
        a, b = _cdict(c0), _cdict(c1)
        for k in ("prim_quartets", "class_prim_quartets", "culled_bound_ledger"):
            a.pop(k), b.pop(k)
        assert a == b
        assert c1.culled_bound_ledger == pytest.approx(c0.culled_bound_ledger, rel=1e-13)
        assert c1.prim_quartets < c0.prim_quartets          # the collapse removed primitive quartets
        assert float((K1 - K0).abs().max()) <= 1e-13 * max(1.0, float(K0.abs().max()))
