"""GPU parity: the CUDA path (through the drop-in API and the C ABI) against
the reference's golden vectors and the CPU oracle.

Bar (BASELINE.json north star): identical culled quartet set and counters
(integer work is bit-exact; the only admissible difference is a bound within
1e-12 relative of tau, which the device counts as a tie), K within 1e-10
max-abs in FP64 (observed ~1e-15), culled-bound ledger within 1e-12 relative
(it is an order-dependent FP64 sum in the reference too).
"""

import numpy as np
import pytest

import paper_1401_6961_b200 as hx
from conftest import (CASES, counters_vec, quartet_bits, system_from_arrays, tree_walk)
from oracle import hexfock_oracle as ho
from paper_1401_6961_b200 import configs

pytestmark = pytest.mark.gpu

FIXTURES = ["cluster1", "cluster3", "cluster5", "cluster10", "ragged0", "ragged1",
            "ragged2", "ragged3", "identity3", "c1",
            # boundary edges (tests/golden/make_golden.py golden_boundary): leaf spans of
            # up to 16 / 32 shells (the unstaged screen) and the overlap_matrix override
            "leaf16", "leaf32", "ovlp_override"]
K_TOL = 1e-10


def _device_setup(g):
    system = system_from_arrays(g["centers"], g["prims"], g["nprim"])
    leaf = int(g["leaf_size"]) if "leaf_size" in g else 10
    tau_ovlp = float(g["tau_ovlp"]) if "tau_ovlp" in g else 1e-11
    part = hx.build_partition(system, leaf_size=leaf)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=tau_ovlp, overlap_matrix=g.get("S"))
    P_tree = hx.build_matrix_tree(g["P"], part)
    return system, pairs, P_tree


def test_subtree_start_matches_reference(golden):
    """A diagonal subtree as bra = ket = P (the reference accepts any node with
    one shared span, exchange_naive.py:105-108): counters, ledger, evaluated
    set and K (the span's block) equal the reference's at depths 1 and 2."""
    g = golden("subtree")
    system, pairs, P_tree = _device_setup(g)
    keys = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_counters")})
    assert len(keys) == 8
    for key in keys:
        depth, drv, tag = key.split("_")
        b, p = pairs, P_tree
        for _ in range(int(depth[1:])):
            b, p = b.children[(0, 0)], p.children[(0, 0)]
        sym = drv == "sym"
        log = []
        if sym:
            K, c = hx.build_exchange_symmetric(b, p, float(tag), quartet_log=log)
        else:
            K, c = hx.build_exchange_naive(b, b, p, float(tag), quartet_log=log)
        assert K.shape == g[key + "_K"].shape, key
        assert np.array_equal(counters_vec(c, sym), g[key + "_counters"]), key
        assert c.culled_bound_ledger == pytest.approx(float(g[key + "_ledger"]), rel=1e-12, abs=1e-300)
        assert np.abs(K - g[key + "_K"]).max() <= K_TOL, key
        assert np.array_equal(np.asarray(sorted(log), dtype=np.int64).reshape(-1, 4), g[key + "_log"]), key


def test_leaf_spans_above_ten_shells_use_unstaged_screen():
    """leaf_size 32 on a p-shell cube: spans of > 10 shells take the unstaged
    screen; the eightfold driver is supported there too and its K equals the
    fourfold K."""
    cfg = configs.cube_cluster(6, 3, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=32)
    assert max(s.shell_hi - s.shell_lo for s in part.leaves) > 10
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    st = ho.Setup(cfg.system, cfg.P, tau_ovlp=1e-11, leaf_size=32)
    K4, c4 = hx.build_exchange_symmetric(pairs, P_tree, 1e-8)
    K4r, c4r = st.symmetric(1e-8)
    assert np.array_equal(counters_vec(c4, True), counters_vec(c4r, True))
    assert np.abs(K4 - K4r).max() <= K_TOL
    K8, _ = hx.build_exchange_eightfold(pairs, P_tree, 1e-8)
    assert np.abs(K8 - K4).max() <= 1e-12


@pytest.mark.parametrize("name", FIXTURES)
def test_device_trees_match_reference(golden, name):
    g = golden(name)
    _, pairs, P_tree = _device_setup(g)
    pw = np.array(tree_walk(pairs))
    ref = g["pair_walk"]
    assert pw.shape == ref.shape
    assert np.array_equal(pw[:, :5], ref[:, :5])            # spans
    assert np.array_equal(pw[:, 6], ref[:, 6])              # pruned flags
    assert np.allclose(pw[:, 5], ref[:, 5], rtol=1e-13, atol=0)   # diag norms (device Q)
    assert np.allclose(pw[:, 7:], ref[:, 7:], rtol=1e-13, atol=0)
    mw = np.array(tree_walk(P_tree))
    assert np.array_equal(mw[:, :6], g["p_walk"][:, :6])    # fsum norms: bitwise


@pytest.mark.parametrize("name", FIXTURES)
def test_device_drivers_match_reference(golden, name):
    g = golden(name)
    system, pairs, P_tree = _device_setup(g)
    n_sh = system.n_shells
    keys = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_counters")})
    for key in keys:
        sym = key.startswith("sym")
        tag = key.split("_", 1)[1]
        mode = "literal" if tag == "literal" else "schwarz"
        tau = 1e-8 if tag == "literal" else float(tag)
        log = [] if key + "_qbits" in g else None
        if sym:
            K, c = hx.build_exchange_symmetric(pairs, P_tree, tau, mode=mode, quartet_log=log)
        else:
            K, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau, mode=mode, quartet_log=log)
        assert c.ties_task == 0 and c.ties_leaf == 0, key
        assert np.array_equal(counters_vec(c, sym), g[key + "_counters"]), key
        assert c.culled_bound_ledger == pytest.approx(float(g[key + "_ledger"]), rel=1e-12, abs=1e-300)
        err = np.abs(K - g[key + "_K"]).max()
        assert err <= K_TOL, (key, err)
        if log is not None:
            bits = quartet_bits(log, n_sh)
            ref = np.unpackbits(g[key + "_qbits"])[:n_sh ** 4].astype(bool)
            assert np.array_equal(bits, ref), key


def _p_case(units, seed, leaf):
    cfg = configs.cube_cluster(units, seed, "tiny")
    return cfg.system, cfg.P, leaf


@pytest.mark.parametrize("units,seed,leaf,tau_ovlp,taus", [
    (2, 9, 4, 0.0, (0.0, 1e-8)),
    (3, 4, 6, 1e-11, (1e-10, 1e-8, 1e-6)),
    (6, 5, 10, 1e-11, (1e-8,)),
])
def test_pshell_parity_with_oracle(units, seed, leaf, tau_ovlp, taus):
    system, P, leaf = _p_case(units, seed, leaf)
    st = ho.Setup(system, P, tau_ovlp=tau_ovlp, leaf_size=leaf)
    part = hx.build_partition(system, leaf_size=leaf)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=tau_ovlp)
    P_tree = hx.build_matrix_tree(P, part)
    for tau in taus:
        for sym in (False, True):
            log, ref_log = [], []
            if sym:
                K, c = hx.build_exchange_symmetric(pairs, P_tree, tau, quartet_log=log)
                K_ref, c_ref = st.symmetric(tau, quartet_log=ref_log)
            else:
                K, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau, quartet_log=log)
                K_ref, c_ref = st.naive(tau, quartet_log=ref_log)
            assert c.ties_task == 0 and c.ties_leaf == 0
            assert np.array_equal(counters_vec(c, sym), counters_vec(c_ref, sym)), (tau, sym)
            assert set(log) == set(ref_log)
            assert c.culled_bound_ledger == pytest.approx(c_ref.culled_bound_ledger, rel=1e-12, abs=1e-300)
            assert np.abs(K - K_ref).max() <= K_TOL


def test_pshell_dense_oracle_exactness():
    system, P, leaf = _p_case(2, 9, 4)
    st = ho.Setup(system, P, tau_ovlp=0.0, leaf_size=leaf)
    K_dense = ho.dense_exchange(st.shells, P)
    part = hx.build_partition(system, leaf_size=leaf)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=0.0)
    P_tree = hx.build_matrix_tree(P, part)
    K_n, _ = hx.build_exchange_naive(pairs, pairs, P_tree, 0.0)
    K_s, _ = hx.build_exchange_symmetric(pairs, P_tree, 0.0)
    assert np.abs(K_n - K_dense).max() <= 1e-12
    assert np.abs(K_s - K_dense).max() <= 1e-12


def test_repeated_builds_bitwise_identical():
    cfg = configs.cube_cluster(4, 7, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=6)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    for f in (lambda: hx.build_exchange_naive(pairs, pairs, P_tree, 1e-9),
              lambda: hx.build_exchange_symmetric(pairs, P_tree, 1e-9)):
        K1, c1 = f()
        K2, c2 = f()
        assert np.array_equal(K1, K2)
        assert c1.to_dict() == c2.to_dict()


@pytest.mark.parametrize("sym", [False, True, "eightfold"])
def test_sharded_shards_sum_to_full_build(sym):
    """Multi-GPU semantics on one device: the shards of a frontier cut, run one
    after another, sum (K and counters) to the unsharded build."""
    from paper_1401_6961_b200 import distributed, exchange
    cfg = configs.cube_cluster(8, 3, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=6)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    K_full, c_full, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-9, "schwarz", sym)
    import torch
    scratch = torch.empty(K_full.shape, dtype=torch.float64, device="cuda")
    for world, strategy in ((2, "balanced"), (3, "balanced"), (2, "hashed"), (3, "hashed"),
                            (2, "cyclic"), (3, "cyclic"), (2, "contiguous"), (3, "contiguous")):
        level, ranges = distributed.plan(pairs, pairs, P_tree, 1e-9, "schwarz", sym, world,
                                         min_tasks_per_rank=4, strategy=strategy, K_scratch=scratch,
                                         groups_per_rank=4)
        K = np.zeros_like(K_full)
        vec = 0
        for b, e, s in ranges:
            Ks, c, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-9, "schwarz", sym,
                                             shard=(level, b, e, s), symmetrize=False)
            K += Ks
            vec = vec + distributed.counters_vector(c)
        if sym is True:
            K = hx.symmetrize_final(K)
        full = distributed.counters_vector(c_full)
        assert np.array_equal(vec[:-1], full[:-1]), (world, level, ranges)
        assert vec[-1] == pytest.approx(full[-1], rel=1e-12)
        assert np.abs(K - K_full).max() <= 1e-13
        # the multi-GPU reduction path: integer sum of the shards' fixed-point
        # accumulators (one scale for all shards) is bitwise the unsharded K
        import torch
        n = K_full.shape[0]
        acc, scales = None, set()
        for b, e, s in ranges:
            buf = torch.empty((n, n), dtype=torch.int64, device="cuda")
            (kf, S), _, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-9, "schwarz", sym,
                                                  shard=(level, b, e, s), symmetrize=False,
                                                  K_out=buf, K_fixed=True)
            scales.add(S)
            acc = kf.clone() if acc is None else acc + kf
        assert len(scales) == 1
        Kx = torch.empty((n, n), dtype=torch.float64, device="cuda")
        from paper_1401_6961_b200 import _native
        import ctypes
        _native.check(_native.lib().hxf_fixed_to_double(ctypes.c_void_p(acc.data_ptr()), acc.numel(),
                                                        scales.pop(), ctypes.c_void_p(Kx.data_ptr()),
                                                        _native.current_stream()))
        Kx = Kx.cpu().numpy()
        if sym is True:
            Kx = hx.symmetrize_final(Kx)
        assert np.array_equal(Kx, K_full), np.abs(Kx - K_full).max()


@pytest.mark.gpu
@pytest.mark.parametrize("sym", [False, True])
def test_primitive_neglect_within_bound(sym, monkeypatch):
    """Per-build primitive neglect (HXF_PRIM_EPS): dropping primitive
    pairs with S_ab * max S_cd * max|P| <= eps changes K by at most eps per
    dropped primitive quartet, leaves the culled set (counters) unchanged, and
    eps = 0 keeps every primitive."""
    from paper_1401_6961_b200 import exchange
    cfg = configs.cube_cluster(12, 5, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=8)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    monkeypatch.setenv("HXF_PRIM_EPS", "0")
    K0, c0, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-8, "schwarz", sym)
    full = sum(int(x) for x in c0.class_prim_quartets)
    monkeypatch.setenv("HXF_PRIM_EPS", "1e-9")   # coarse threshold: many primitives dropped
    K1, c1, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-8, "schwarz", sym)
    kept = sum(int(x) for x in c1.class_prim_quartets)
    assert c1.eri_shell_quartets == c0.eri_shell_quartets
    assert c1.quartets_culled_leaf == c0.quartets_culled_leaf
    assert kept < full
    # each dropped primitive quartet changes an element by <= eps per function
    # component of the contracted density block (<= 9) in each of <= 4 slots
    assert np.abs(K1 - K0).max() <= 36 * 1e-9 * (full - kept)
    monkeypatch.delenv("HXF_PRIM_EPS")
    K2, c2, _ = exchange.run_exchange(pairs, pairs, P_tree, 1e-8, "schwarz", sym)
    assert sum(int(x) for x in c2.class_prim_quartets) <= full
    assert np.abs(K2 - K0).max() <= 1e-12


def _fold(log):
    """4-fold quartet tuples folded bra <-> ket: {min((i,j,k,l), (k,l,i,j))}."""
    return {min((i, j, k, l), (k, l, i, j)) for (i, j, k, l) in log}


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["s_lattice", "p_cube"])
def test_eightfold_matches_fourfold(case):
    """Eightfold mode (optional): evaluated set = the 4-fold
    quartet log folded to unordered (bra pair, ket pair); K equal to the 4-fold
    K within rounding; about half the quartets."""
    if case == "s_lattice":
        cfg = configs.config1()
        leaf = 4
    else:
        cfg = configs.cube_cluster(10, 7, "tiny")
        leaf = 6
    part = hx.build_partition(cfg.system, leaf_size=leaf)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    log4, log8 = [], []
    K4, c4 = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=1e-8, quartet_log=log4)
    K8, c8 = hx.build_exchange_eightfold(pairs, P_tree, tau_2e=1e-8, quartet_log=log8)
    assert c4.ties_leaf == 0 and c8.ties_leaf == 0 and c8.ties_task == 0
    # each unordered (bra pair, ket pair) exactly once, and exactly the folded 4-fold set
    assert len(log8) == len(_fold(log8)) == c8.eri_shell_quartets
    assert _fold(log8) == _fold(log4)
    assert np.array_equal(K8, K8.T)
    assert np.abs(K8 - K4).max() <= 1e-12
    assert c8.eri_shell_quartets < 0.6 * c4.eri_shell_quartets


def test_ss_eri_precision_c1(golden):
    """(ss|ss)-only config 1 against the reference's own K at tau = 1e-8: with the
    identical culled set the difference is FP64 rounding only (the (ss|ss) kernel's
    fine-grid F_0, boys_f0_fine, T from 0 past the asymptotic switch)."""
    g = golden("c1")
    _, pairs, P_tree = _device_setup(g)
    for key, f in (("naive_1e-08", lambda: hx.build_exchange_naive(pairs, pairs, P_tree, 1e-8)),
                   ("sym_1e-08", lambda: hx.build_exchange_symmetric(pairs, P_tree, 1e-8))):
        K, _ = f()
        err = np.abs(K - g[key + "_K"]).max()
        assert err <= 5e-14, (key, err)


def test_scratch_release_between_builds():
    """Cached build scratch can be handed back; the next build is unchanged."""
    cfg = configs.cube_cluster(4, 3, "tiny")
    part = hx.build_partition(cfg.system, leaf_size=6)
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    K1, c1 = hx.build_exchange_symmetric(pairs, P_tree, 1e-9)
    assert hx.release_scratch() > 0
    assert hx.release_scratch() == 0
    K2, c2 = hx.build_exchange_symmetric(pairs, P_tree, 1e-9)
    assert np.array_equal(K1, K2) and c1.to_dict() == c2.to_dict()


@pytest.mark.parametrize("sym", [False, True])
@pytest.mark.parametrize("case", ["single_leaf", "cut_below_frontier"])
def test_shards_above_unreached_cut_hold_no_work(sym, case):
    """A shard with shard_begin != 0 whose cut level is never reached (a single
    leaf span, or a cut deeper than where the frontier empties) owns no leaf task:
    the shards still sum to the unsharded build (traverse.cu)."""
    from paper_1401_6961_b200 import exchange
    if case == "single_leaf":
        cfg = configs.cube_cluster(1, 3, "one")
        part = hx.build_partition(cfg.system, leaf_size=10)
        assert len(part.levels) == 1
        level, tau = 0, 1e-8
    else:
        cfg = configs.cube_cluster(8, 3, "tiny")
        part = hx.build_partition(cfg.system, leaf_size=6)
        level, tau = len(part.levels) + 3, 1e-9     # the traversal ends above this cut
    pairs = hx.build_pair_tree(cfg.system, part, tau_ovlp=1e-11)
    P_tree = hx.build_matrix_tree(cfg.P, part)
    K_full, c_full, _ = exchange.run_exchange(pairs, pairs, P_tree, tau, "schwarz", sym, symmetrize=False)
    K0, c0, _ = exchange.run_exchange(pairs, pairs, P_tree, tau, "schwarz", sym, shard=(level, 0, 1 << 20),
                                      symmetrize=False)
    K1, c1, _ = exchange.run_exchange(pairs, pairs, P_tree, tau, "schwarz", sym, shard=(level, 1, 1 << 20),
                                      symmetrize=False)
    assert not np.any(K1)
    assert c1.eri_shell_quartets == 0 and c1.leaf_contractions == 0
    assert np.array_equal(K0 + K1, K_full)
    assert c0.eri_shell_quartets == c_full.eri_shell_quartets
