"""Generate golden vectors by running the REFERENCE implementation.

Run in the build container only (the reference does not exist on GPU boxes):

    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Each file pins one behaviour of the reference's
hot path (counters, culled quartet sets, tree norms, K) on a seeded input;
tests/test_oracle_golden.py checks the CPU oracle against them and the GPU
parity tests check the CUDA path against the oracle and these fixtures.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

import hexfock  # noqa: E402  (the reference)
from hexfock import basis as rb  # noqa: E402
from hexfock import integrals as ri  # noqa: E402
from hexfock import quadtree as rq  # noqa: E402
from hexfock.exchange_naive import build_exchange_naive  # noqa: E402
from hexfock.exchange_symmetry import build_exchange_symmetric  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1401_6961_b200 import configs  # noqa: E402

COUNTER_KEYS = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
                "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
                "tasks_expanded", "children_spawned")
SYM_KEYS = ("links_culled_screening", "links_culled_absent")
CASES = ("A", "B", "C", "D", "E", "F1", "F2", "H", "SPARSE")


def walk(node, level=0, out=None):
    out = [] if out is None else out
    norm = getattr(node, "norm", None)
    if norm is None:
        norm = node.diag_norm
    out.append((level, node.row.fn_lo, node.row.fn_hi, node.col.fn_lo, node.col.fn_hi,
                norm, float(getattr(node, "pruned", False)),
                getattr(node, "rowsum_max", 0.0), getattr(node, "colsum_max", 0.0)))
    for key in sorted(getattr(node, "children", {}) or {}):
        walk(node.children[key], level + 1, out)
    return out


def counters_vec(c, sym):
    v = [getattr(c, k) for k in COUNTER_KEYS]
    if sym:
        v += [getattr(c, k) for k in SYM_KEYS]
        v += [c.case_tasks[k] for k in CASES] + [c.case_leaf_tasks[k] for k in CASES]
    return np.asarray(v, dtype=np.int64)


def system_arrays(system):
    centers = np.array([sh.center for sh in system.shells])
    prims = [np.array(sh.primitives, dtype=float) for sh in system.shells]
    nprim = np.array([len(p) for p in prims])
    return centers, np.concatenate(prims), nprim


def ref_system_from(cfg_system):
    shells = [rb.GaussianShell(center=sh.center.copy(), primitives=list(sh.primitives))
              for sh in cfg_system.shells]
    for k, sh in enumerate(shells):
        sh.function_offset = k
    return rb.BasisSystem(shells=shells, atoms=[])


def run_drivers(system, pairs, P_tree, taus, out, log_taus=(), mode="schwarz"):
    n_sh = system.n_shells
    for tau in taus:
        tag = f"{tau:g}"
        for sym in (False, True):
            log = [] if tau in log_taus else None
            if sym:
                K, c = build_exchange_symmetric(pairs, P_tree, tau, mode=mode, quartet_log=log)
            else:
                K, c = build_exchange_naive(pairs, pairs, P_tree, tau, mode=mode, quartet_log=log)
            pre = ("sym" if sym else "naive") + "_" + tag
            out[pre + "_K"] = K
            out[pre + "_counters"] = counters_vec(c, sym)
            out[pre + "_ledger"] = np.float64(c.culled_bound_ledger)
            if log is not None:
                bits = np.zeros(n_sh ** 4, dtype=bool)
                arr = np.asarray(log, dtype=np.int64).reshape(-1, 4)
                flat = ((arr[:, 0] * n_sh + arr[:, 1]) * n_sh + arr[:, 2]) * n_sh + arr[:, 3]
                assert len(np.unique(flat)) == len(flat)
                bits[flat] = True
                out[pre + "_qbits"] = np.packbits(bits)


def save(name, out):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


def golden_clusters():
    # conftest.build_setup restated: generate_cluster -> hilbert_order ->
    # partition -> pair tree -> default exp-decay density (conftest.py:22-36)
    for n, tau_ovlp, taus, log_taus in ((1, 0.0, (0.0, 1e-8), (0.0,)),
                                        (3, 0.0, (0.0, 1e-10, 1e-8, 1e-6), (1e-8,)),
                                        (5, 1e-11, (0.0, 1e-10, 1e-8), (1e-8,)),
                                        (10, 0.0, (1e-8,), (1e-8,))):
        system = rb.generate_cluster(n, seed=3)
        system, perm = rb.hilbert_order(system)
        part = rq.build_partition(system, leaf_size=10)
        pairs = rq.build_pair_tree(system, part, tau_ovlp=tau_ovlp)
        P = hexfock.build_density(system, hexfock.DensityModel())
        P_tree = rq.build_matrix_tree(P, part)
        centers, prims, nprim = system_arrays(system)
        out = {"centers": centers, "prims": prims, "nprim": nprim, "perm": perm, "P": P,
               "tau_ovlp": np.float64(tau_ovlp), "pair_walk": np.array(walk(pairs)),
               "p_walk": np.array(walk(P_tree)),
               "diag_root": pairs.diag if pairs.is_leaf else np.zeros(0)}
        run_drivers(system, pairs, P_tree, taus, out, log_taus)
        if n == 3:
            for tau in (1e-8,):
                for sym in (False, True):
                    f = build_exchange_symmetric if sym else build_exchange_naive
                    args = (pairs, P_tree) if sym else (pairs, pairs, P_tree)
                    K, c = f(*args, tau, mode="literal")
                    pre = ("sym" if sym else "naive") + "_literal"
                    out[pre + "_K"] = K
                    out[pre + "_counters"] = counters_vec(c, sym)
                    out[pre + "_ledger"] = np.float64(c.culled_bound_ledger)
        save(f"cluster{n}", out)


def golden_c1():
    cfg = configs.config1()
    system = ref_system_from(cfg.system)
    part = rq.build_partition(system, leaf_size=10)
    pairs = rq.build_pair_tree(system, part, tau_ovlp=cfg.tau_ovlp)
    P_tree = rq.build_matrix_tree(cfg.P, part)
    centers, prims, nprim = system_arrays(system)
    out = {"centers": centers, "prims": prims, "nprim": nprim, "P": cfg.P,
           "pair_walk": np.array(walk(pairs)), "p_walk": np.array(walk(P_tree))}
    run_drivers(system, pairs, P_tree, (cfg.tau_2e,), out, (cfg.tau_2e,))
    save("c1", out)


def line_system(n, rng):
    shells = []
    for i in range(n):
        k = int(rng.integers(1, 3))
        prims = list(zip(rng.uniform(0.3, 3.0, k), rng.uniform(0.2, 1.0, k)))
        shells.append(rb.GaussianShell(center=[i * 1.1, 0.3 * (i % 3), 0.0], primitives=prims))
    for i, sh in enumerate(shells):
        sh.function_offset = i
    return rb.BasisSystem(shells=shells, atoms=[])


def golden_ragged():
    # ragged partitions + zero blocks (absent P links, SPARSE) in the style of
    # test_acceptance.py:208-235
    rng = np.random.default_rng(4242)
    for t, (n, leaf) in enumerate(((13, 4), (21, 3), (27, 5), (9, 2))):
        system = line_system(n, rng)
        part = rq.build_partition(system, leaf_size=leaf)
        pairs = rq.build_pair_tree(system, part, tau_ovlp=1e-9)
        P = rng.normal(size=(n, n))
        P = 0.5 * (P + P.T)
        P[rng.random(size=P.shape) < 0.5] = 0.0
        P = np.triu(P) + np.triu(P, 1).T
        P[:3, n - 4:] = 0.0
        P[n - 4:, :3] = 0.0
        P_tree = rq.build_matrix_tree(P, part)
        centers, prims, nprim = system_arrays(system)
        out = {"centers": centers, "prims": prims, "nprim": nprim, "P": P,
               "leaf_size": np.int64(leaf), "tau_ovlp": np.float64(1e-9),
               "pair_walk": np.array(walk(pairs)), "p_walk": np.array(walk(P_tree))}
        run_drivers(system, pairs, P_tree, (0.0, 1e-4), out, (0.0, 1e-4))
        save(f"ragged{t}", out)
    # identity density: SPARSE demotion (test_exchange_symmetry.py:105-118)
    system = rb.generate_cluster(3, seed=3)
    part = rq.build_partition(system)
    pairs = rq.build_pair_tree(system, part, tau_ovlp=0.0)
    P = np.eye(system.n_functions)
    P_tree = rq.build_matrix_tree(P, part)
    centers, prims, nprim = system_arrays(system)
    out = {"centers": centers, "prims": prims, "nprim": nprim, "P": P,
           "tau_ovlp": np.float64(0.0), "pair_walk": np.array(walk(pairs)),
           "p_walk": np.array(walk(P_tree))}
    run_drivers(system, pairs, P_tree, (0.0,), out, (0.0,))
    save("identity3", out)


def golden_integrals():
    rng = np.random.default_rng(2024)
    t = np.concatenate([np.linspace(0.0, 50.0, 2001), [11.999999, 12.0, 12.000001, 1e-12, 300.0]])
    out = {"boys_t": t, "boys_f0": ri.boys_f0(t)}
    quartets, vals = [], []
    for _ in range(40):
        shells = []
        for _ in range(4):
            k = int(rng.integers(1, 4))
            shells.append(rb.GaussianShell(center=rng.normal(scale=2.5, size=3),
                                           primitives=list(zip(rng.uniform(0.1, 30.0, k),
                                                               rng.uniform(0.2, 1.0, k)))))
        vals.append(ri.eri_quartet(*shells).values[0, 0, 0, 0])
        rec = []
        for sh in shells:
            pr = np.zeros((3, 2))
            pr[:len(sh.primitives)] = sh.primitives
            rec.append(np.concatenate([sh.center, [len(sh.primitives)], pr.ravel()]))
        quartets.append(np.stack(rec))
    out["eri_shells"] = np.stack(quartets)
    out["eri_values"] = np.array(vals)
    ov = []
    for _ in range(40):
        a = rb.GaussianShell(center=rng.normal(scale=1.5, size=3),
                             primitives=[(float(rng.uniform(0.1, 5)), 1.0)])
        b = rb.GaussianShell(center=rng.normal(scale=1.5, size=3),
                             primitives=[(float(rng.uniform(0.1, 5)), 0.7), (2.0, 0.3)])
        ov.append(np.concatenate([a.center, b.center, a.primitives[0],
                                  np.ravel(b.primitives), [ri.overlap(a, b)]]))
    out["overlaps"] = np.array(ov)
    geo = []
    for n, seed in ((5, 3), (12, 7), (30, 11)):
        s = rb.generate_cluster(n, seed=seed)
        s2, perm = rb.hilbert_order(s)
        geo.append((n, seed, np.array([sh.center for sh in s.shells]), perm))
    for k, (n, seed, c, perm) in enumerate(geo):
        out[f"geo{k}_n"] = np.int64(n)
        out[f"geo{k}_seed"] = np.int64(seed)
        out[f"geo{k}_centers"] = c
        out[f"geo{k}_perm"] = perm
    save("integrals", out)


def golden_boundary():
    """Reference behaviours at the edges of the drop-in boundary: leaf spans
    above 10 shells (--leaf-size accepts any value, cli.py:289), the
    overlap_matrix override of build_pair_tree (quadtree.py:284-293) and a
    diagonal subtree as the start node (any bra/ket/P with one shared span,
    exchange_naive.py:105-108)."""
    for leaf in (16, 32):
        system = rb.generate_cluster(20, seed=5)
        system, perm = rb.hilbert_order(system)
        part = rq.build_partition(system, leaf_size=leaf)
        pairs = rq.build_pair_tree(system, part, tau_ovlp=1e-11)
        P = hexfock.build_density(system, hexfock.DensityModel())
        P_tree = rq.build_matrix_tree(P, part)
        centers, prims, nprim = system_arrays(system)
        out = {"centers": centers, "prims": prims, "nprim": nprim, "P": P,
               "leaf_size": np.int64(leaf), "tau_ovlp": np.float64(1e-11),
               "pair_walk": np.array(walk(pairs)), "p_walk": np.array(walk(P_tree))}
        run_drivers(system, pairs, P_tree, (0.0, 1e-8), out, (1e-8,))
        save(f"leaf{leaf}", out)
    # overlap_matrix override: a non-symmetric |S| (computed overlaps times a
    # seeded factor in [0.01, 3]) prunes a different set of nodes
    rng = np.random.default_rng(77)
    system = rb.generate_cluster(8, seed=9)
    system, _ = rb.hilbert_order(system)
    part = rq.build_partition(system, leaf_size=4)
    S = rq.shell_overlap_matrix(system) * rng.uniform(0.01, 3.0, size=(system.n_shells,) * 2)
    pairs = rq.build_pair_tree(system, part, tau_ovlp=1e-3, overlap_matrix=S)
    P = hexfock.build_density(system, hexfock.DensityModel())
    P_tree = rq.build_matrix_tree(P, part)
    centers, prims, nprim = system_arrays(system)
    out = {"centers": centers, "prims": prims, "nprim": nprim, "P": P, "S": S,
           "leaf_size": np.int64(4), "tau_ovlp": np.float64(1e-3),
           "pair_walk": np.array(walk(pairs)), "p_walk": np.array(walk(P_tree))}
    run_drivers(system, pairs, P_tree, (0.0, 1e-8), out, (1e-8,))
    save("ovlp_override", out)
    # diagonal subtree start: the root's first (left, left) child and its
    # (left, left) grandchild, spans starting at function 0
    system = rb.generate_cluster(10, seed=3)
    system, _ = rb.hilbert_order(system)
    part = rq.build_partition(system, leaf_size=4)
    pairs = rq.build_pair_tree(system, part, tau_ovlp=1e-11)
    P = hexfock.build_density(system, hexfock.DensityModel())
    P_tree = rq.build_matrix_tree(P, part)
    centers, prims, nprim = system_arrays(system)
    out = {"centers": centers, "prims": prims, "nprim": nprim, "P": P,
           "leaf_size": np.int64(4), "tau_ovlp": np.float64(1e-11)}
    for depth in (1, 2):
        b, p = pairs, P_tree
        for _ in range(depth):
            b, p = b.children[(0, 0)], p.children[(0, 0)]
        for tau in (0.0, 1e-8):
            for sym in (False, True):
                log = []
                if sym:
                    K, c = build_exchange_symmetric(b, p, tau, quartet_log=log)
                else:
                    K, c = build_exchange_naive(b, b, p, tau, quartet_log=log)
                pre = f"d{depth}_" + ("sym" if sym else "naive") + f"_{tau:g}"
                out[pre + "_K"] = K
                out[pre + "_counters"] = counters_vec(c, sym)
                out[pre + "_ledger"] = np.float64(c.culled_bound_ledger)
                out[pre + "_log"] = np.asarray(sorted(log), dtype=np.int64).reshape(-1, 4)
    save("subtree", out)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        for name in sys.argv[1:]:
            globals()["golden_" + name]()
        sys.exit(0)
    golden_integrals()
    golden_ragged()
    golden_clusters()
    golden_c1()
    golden_boundary()
