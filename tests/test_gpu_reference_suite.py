"""The reference's own driver tests (test_exchange_naive.py,
test_exchange_symmetry.py, test_quadtree.py, acceptance criteria 1-5, 9),
restated against the drop-in GPU API.  Dense references come from the CPU
oracle (the checker)."""

import math

import numpy as np
import pytest

import paper_1401_6961_b200 as hx
from oracle import hexfock_oracle as ho

pytestmark = pytest.mark.gpu


def build_setup(n_molecules, seed=3, tau_ovlp=0.0, gamma=None, leaf_size=10, density=None):
    system = hx.generate_cluster(n_molecules, seed=seed)
    system, _ = hx.hilbert_order(system)
    part = hx.build_partition(system, leaf_size=leaf_size)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=tau_ovlp)
    if density is None:
        model = hx.DensityModel() if gamma is None else hx.DensityModel(gamma=gamma)
        P = hx.build_density(system, model)
    else:
        P = np.asarray(density, dtype=float)
    return system, pairs, hx.build_matrix_tree(P, part), P


def dense_K(system, P):
    return ho.dense_exchange(ho.as_oracle_shells(system), P)


# ------------------------------------------------ test_exchange_naive.py

def test_zero_density_yields_zero_exchange():
    system = hx.generate_cluster(2, seed=3)
    part = hx.build_partition(system)
    P_tree = hx.build_matrix_tree(np.zeros((system.n_functions,) * 2), part)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=0.0)
    K, c = hx.build_exchange_naive(pairs, pairs, P_tree)
    assert not np.any(K)
    assert c.leaf_contractions == 0


def test_infinite_threshold_culls_at_root():
    _, pairs, P_tree, _ = build_setup(2)
    K, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=math.inf)
    assert not np.any(K)
    assert c.tasks_visited == 1 and c.tasks_culled_screening == 1 and c.leaf_contractions == 0


def test_negative_tau_and_mode_rejected():
    _, pairs, P_tree, _ = build_setup(1)
    with pytest.raises(hx.InvalidArgumentError):
        hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=-1.0)
    with pytest.raises(hx.InvalidArgumentError):
        hx.build_exchange_symmetric(pairs, P_tree, tau_2e=-1.0)
    with pytest.raises(hx.InvalidArgumentError):
        hx.build_exchange_symmetric(pairs, P_tree, mode="bogus")


def test_partition_mismatch_rejected():
    _, pairs_a, _, _ = build_setup(1)
    system = hx.generate_cluster(1, seed=3)
    part = hx.build_partition(system)
    P_tree = hx.build_matrix_tree(np.eye(system.n_functions), part)
    with pytest.raises(hx.InvalidArgumentError):
        hx.build_exchange_naive(pairs_a, pairs_a, P_tree)


def test_exact_against_dense_oracle():
    for n in (1, 2, 3, 5):
        system, pairs, P_tree, P = build_setup(n, tau_ovlp=0.0)
        K_ref = dense_K(system, P)
        K, _ = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=0.0)
        K_s, _ = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=0.0)
        assert np.abs(K - K_ref).max() <= 1e-11
        assert np.abs(K_s - K_ref).max() <= 1e-11


def test_screened_error_within_culled_bound_ledger_and_monotone():
    system, pairs, P_tree, P = build_setup(5, tau_ovlp=0.0)
    K_exact, _ = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=0.0)
    prev = math.inf
    for tau in (1e-4, 1e-6, 1e-8, 1e-10, 1e-12):
        for f in (lambda t: hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=t),
                  lambda t: hx.build_exchange_symmetric(pairs, P_tree, tau_2e=t)):
            K, c = f(tau)
            err = np.abs(K - K_exact).max()
            assert err <= c.culled_bound_ledger + 1e-15
        e = float(np.linalg.norm(hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=tau)[0] - K_exact))
        assert e <= prev + 1e-15
        prev = e


def test_counter_conservation():
    for n, tau in ((3, 0.0), (5, 1e-8), (5, 1e-6)):
        _, pairs, P_tree, _ = build_setup(n)
        _, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=tau)
        assert c.tasks_visited == (c.tasks_culled_screening + c.tasks_culled_absent
                                   + c.leaf_contractions + c.tasks_expanded)
        assert c.tasks_visited == c.children_spawned + 1
        _, s = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=tau, evaluate=False)
        assert sum(s.case_tasks.values()) == s.leaf_contractions + s.tasks_expanded
        assert sum(s.case_leaf_tasks.values()) == s.leaf_contractions


def test_sequential_determinism_and_threads_argument():
    _, pairs, P_tree, _ = build_setup(3)
    K1, c1 = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=1e-9)
    K2, c2 = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=1e-9, threads=2)
    assert np.array_equal(K1, K2)
    assert c1.to_dict() == c2.to_dict()


def test_evaluate_false_counts_without_integrals():
    _, pairs, P_tree, _ = build_setup(2)
    K, dry = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=1e-9, evaluate=False)
    assert not np.any(K)
    _, wet = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=1e-9)
    assert dry.to_dict() == wet.to_dict()
    log = []
    hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=1e-9, evaluate=False, quartet_log=log)
    assert log == []


def test_quartet_log_collects_evaluated_quartets():
    _, pairs, P_tree, _ = build_setup(1, tau_ovlp=0.0)
    log = []
    _, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=0.0, quartet_log=log)
    assert len(log) == c.eri_shell_quartets and all(len(t) == 4 for t in log)
    log = []
    _, c = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=0.0, quartet_log=log)
    assert len(log) == c.eri_shell_quartets
    assert all(i <= j and k <= l for i, j, k, l in log)


# ------------------------------------------------ test_exchange_symmetry.py

def test_identity_density_sparse_path():
    system = hx.generate_cluster(3, seed=3)
    part = hx.build_partition(system)
    pairs = hx.build_pair_tree(system, part, tau_ovlp=0.0)
    P = np.eye(system.n_functions)
    K, c = hx.build_exchange_symmetric(pairs, hx.build_matrix_tree(P, part), tau_2e=0.0)
    assert np.abs(K - dense_K(system, P)).max() <= 1e-11
    assert c.links_culled_absent > 0 and c.case_tasks["SPARSE"] > 0


def test_raw_accumulator_symmetric():
    _, pairs, P_tree, _ = build_setup(1, tau_ovlp=0.0)
    K, _ = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=0.0)
    assert np.abs(K - K.T).max() == 0.0


def test_canonical_quartet_count_reduction():
    system, pairs, P_tree, _ = build_setup(3, tau_ovlp=0.0)
    _, cn = hx.build_exchange_naive(pairs, pairs, P_tree, tau_2e=0.0, evaluate=False)
    _, cs = hx.build_exchange_symmetric(pairs, P_tree, tau_2e=0.0, evaluate=False)
    ns = system.n_shells
    assert cn.eri_shell_quartets == ns ** 4
    assert cs.eri_shell_quartets == (ns * (ns + 1) // 2) ** 2


def test_naive_symmetric_agreement_grid():
    for tau_ovlp in (0.0, 1e-13, 1e-11):
        _, pairs, P_tree, _ = build_setup(5, tau_ovlp=tau_ovlp)
        for tau in (0.0, 1e-12, 1e-10, 1e-8):
            K_n, _ = hx.build_exchange_naive(pairs, pairs, P_tree, tau)
            K_s, _ = hx.build_exchange_symmetric(pairs, P_tree, tau)
            assert np.abs(K_s - K_n).max() <= 1e-11 * max(1.0, np.abs(K_n).max())


def test_classify_cases_by_span_relation():
    _, pairs, _, _ = build_setup(10, tau_ovlp=0.0)
    lp = lambda i, j: pairs.child(i // 2, j // 2).child(i % 2, j % 2)
    cq = hx.classify_quartet
    assert cq(lp(0, 1), lp(2, 3)).case_id == "A"
    assert cq(lp(0, 0), lp(1, 2)).case_id == "B"
    assert cq(lp(0, 3), lp(1, 2)).case_id == "C"
    assert cq(lp(0, 2), lp(1, 3)).case_id == "D"
    assert cq(lp(0, 1), lp(0, 1)).case_id == "E"
    assert cq(lp(0, 2), lp(0, 3)).case_id == "F1"
    assert cq(lp(0, 2), lp(1, 2)).case_id == "F2"
    assert cq(lp(0, 0), lp(1, 1)).case_id == "H"
    with pytest.raises(hx.LogicError):
        cq(pairs.child(1, 0), pairs.child(1, 1))


# ------------------------------------------------ acceptance 3 and 9

def test_direct_scf_set_identity():
    system, pairs, P_tree, P = build_setup(10, tau_ovlp=0.0)
    log = []
    hx.build_exchange_naive(pairs, pairs, P_tree, 1e-8, quartet_log=log)
    ref = []
    ho.dense_exchange_screened(ho.as_oracle_shells(system), P, 1e-8, quartet_log=ref)
    assert set(log) == set(ref)


def test_random_configs_counter_conservation():
    master = np.random.default_rng(777)
    for seed in master.integers(0, 2 ** 32, 20):
        rng = np.random.default_rng(int(seed))
        _, pairs, P_tree, _ = build_setup(int(rng.integers(1, 3)), seed=int(seed) % 100,
                                          tau_ovlp=10.0 ** rng.uniform(-13, -9))
        tau = 10.0 ** rng.uniform(-12.0, -4.0)
        _, c = hx.build_exchange_naive(pairs, pairs, P_tree, tau, evaluate=False)
        assert c.tasks_visited == (c.tasks_culled_screening + c.tasks_culled_absent
                                   + c.leaf_contractions + c.tasks_expanded)
        _, s = hx.build_exchange_symmetric(pairs, P_tree, tau, evaluate=False)
        assert s.tasks_visited == (s.tasks_culled_screening + s.tasks_culled_absent
                                   + s.leaf_contractions + s.tasks_expanded)


# ------------------------------------------------ test_quadtree.py

def test_matrix_tree_views():
    shells = [hx.GaussianShell(center=[i, 0.0, 0.0], primitives=[(1.0, 1.0)]) for i in range(40)]
    from paper_1401_6961_b200.basis import assign_offsets
    system = hx.BasisSystem(shells=assign_offsets(shells), atoms=[])
    part = hx.build_partition(system, leaf_size=7)
    m = np.random.default_rng(17).normal(size=(40, 40))
    tree = hx.build_matrix_tree(m, part)
    assert np.array_equal(tree.dense(), m)
    t = hx.transpose_view(tree)
    assert np.array_equal(t.dense(), m.T) and hx.transpose_view(t) is tree
    z = hx.build_matrix_tree(np.zeros((40, 40)), part)
    assert z.norm == 0.0 and not z.children
    with pytest.raises(hx.InvalidArgumentError):
        hx.build_matrix_tree(np.zeros((11, 11)), part)


def test_pair_tree_far_clusters_pruned():
    shells = [hx.GaussianShell(center=[i, 0.0, 0.0], primitives=[(1.0, 1.0)]) for i in range(8)]
    shells += [hx.GaussianShell(center=[100.0 + i, 0.0, 0.0], primitives=[(1.0, 1.0)]) for i in range(8)]
    from paper_1401_6961_b200.basis import assign_offsets
    system = hx.BasisSystem(shells=assign_offsets(shells), atoms=[])
    part = hx.build_partition(system, leaf_size=8)
    tree = hx.build_pair_tree(system, part, tau_ovlp=1e-13)
    assert tree.child(0, 1).pruned and tree.child(1, 0).pruned
    assert not tree.child(0, 0).pruned and not tree.child(1, 1).pruned


def test_pair_tree_leaf_diag_matches_quartets():
    system, pairs, _, _ = build_setup(1, tau_ovlp=0.0)
    assert pairs.is_leaf
    sh = ho.as_oracle_shells(system)
    for i in range(system.n_shells):
        for j in range(system.n_shells):
            a, b = min(i, j), max(i, j)
            pd = ho.Pairs(sh, [(a, b)])
            ref = ho.ss_cross(pd, pd)[0, 0]
            assert pairs.diag[i, j] == pytest.approx(ref, rel=1e-12)
