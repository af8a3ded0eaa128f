"""Pin the CPU oracle against golden vectors written by the reference.

CPU-only.  Everything the GPU parity tests compare against flows through the
oracle, so this is the link from the CUDA path back to the reference.
"""

import math

import numpy as np
import pytest

from conftest import (CASES, counters_vec, quartet_bits, system_from_arrays, tree_walk)
from oracle import hexfock_oracle as ho
from paper_1401_6961_b200 import basis, configs, inputs

FIXTURES = ["cluster1", "cluster3", "cluster5", "cluster10", "ragged0", "ragged1",
            "ragged2", "ragged3", "identity3", "c1"]


def _setup(g):
    system = system_from_arrays(g["centers"], g["prims"], g["nprim"])
    leaf = int(g["leaf_size"]) if "leaf_size" in g else 10
    tau_ovlp = float(g["tau_ovlp"]) if "tau_ovlp" in g else 1e-11
    return system, ho.Setup(system, g["P"], tau_ovlp=tau_ovlp, leaf_size=leaf)


@pytest.mark.parametrize("name", FIXTURES)
def test_tree_norms_bitwise(golden, name):
    g = golden(name)
    _, st = _setup(g)
    pw = np.array(tree_walk(st.pairs))
    assert pw.shape == g["pair_walk"].shape
    # spans, pruned flags and fsum norms bit-identical; ledger sums to 1e-15
    assert np.array_equal(pw[:, :7], g["pair_walk"][:, :7])
    assert np.allclose(pw[:, 7:], g["pair_walk"][:, 7:], rtol=1e-15, atol=0)
    mw = np.array(tree_walk(st.Ptree))
    assert np.array_equal(mw[:, :6], g["p_walk"][:, :6])


@pytest.mark.parametrize("name", FIXTURES)
def test_drivers_match_reference(golden, name):
    g = golden(name)
    system, st = _setup(g)
    n_sh = system.n_shells
    keys = sorted({k.rsplit("_", 1)[0] for k in g if k.endswith("_counters")})
    assert keys
    for key in keys:
        sym = key.startswith("sym")
        tag = key.split("_", 1)[1]
        mode = "literal" if tag == "literal" else "schwarz"
        tau = 1e-8 if tag == "literal" else float(tag)
        log = [] if key + "_qbits" in g else None
        f = st.symmetric if sym else st.naive
        K, c = f(tau, mode=mode, quartet_log=log)
        assert np.array_equal(counters_vec(c, sym), g[key + "_counters"]), key
        assert c.culled_bound_ledger == pytest.approx(float(g[key + "_ledger"]), rel=1e-12, abs=0)
        assert np.abs(K - g[key + "_K"]).max() <= 1e-13, key
        if log is not None:
            bits = quartet_bits(log, n_sh)
            ref = np.unpackbits(g[key + "_qbits"])[:n_sh ** 4].astype(bool)
            assert np.array_equal(bits, ref), key


@pytest.mark.parametrize("name", ["leaf16", "leaf32"])
def test_large_leaf_spans_match_reference(golden, name):
    """Leaf spans of up to 16 / 32 shells (the reference's --leaf-size takes any
    value): tree, counters, ledger, K and the evaluated set at tau = 1e-8 (the
    tau = 0 keys are checked on the GPU only: the oracle needs minutes there)."""
    g = golden(name)
    system, st = _setup(g)
    pw = np.array(tree_walk(st.pairs))
    assert np.array_equal(pw[:, :7], g["pair_walk"][:, :7])
    n_sh = system.n_shells
    for sym in (False, True):
        key = ("sym" if sym else "naive") + "_1e-08"
        log = []
        K, c = (st.symmetric if sym else st.naive)(1e-8, quartet_log=log)
        assert np.array_equal(counters_vec(c, sym), g[key + "_counters"]), key
        assert c.culled_bound_ledger == pytest.approx(float(g[key + "_ledger"]), rel=1e-12, abs=0)
        assert np.abs(K - g[key + "_K"]).max() <= 1e-13, key
        assert np.array_equal(quartet_bits(log, n_sh), np.unpackbits(g[key + "_qbits"])[:n_sh ** 4].astype(bool))


def test_c1_fold_identity(golden):
    # the 4-fold set is the canonical image of the naive set
    g = golden("c1")
    n = round(len(g["centers"]))
    naive = np.unpackbits(g["naive_1e-08_qbits"])[:n ** 4].astype(bool).reshape((n,) * 4)
    sym = np.unpackbits(g["sym_1e-08_qbits"])[:n ** 4].astype(bool).reshape((n,) * 4)
    canon = np.zeros_like(naive)
    i, j, k, l = np.nonzero(naive)
    canon[np.minimum(i, j), np.maximum(i, j), np.minimum(k, l), np.maximum(k, l)] = True
    assert np.array_equal(canon, sym)


def test_c1_input_regenerates_identically(golden):
    g = golden("c1")
    cfg = configs.config1()
    assert np.array_equal(np.array([sh.center for sh in cfg.system.shells]), g["centers"])
    assert np.array_equal(cfg.P, g["P"])


def test_boys_and_eri_pins(golden):
    g = golden("integrals")
    assert np.array_equal(ho.boys_f0(g["boys_t"]), g["boys_f0"])
    for rec, ref in zip(g["eri_shells"], g["eri_values"]):
        shells = []
        for s in rec:
            k = int(s[3])
            prims = [tuple(x) for x in s[4:].reshape(3, 2)[:k]]
            shells.append(ho.OShell(s[:3], prims))
        bra = ho.Pairs(shells, [(0, 1)])
        ket = ho.Pairs(shells, [(2, 3)])
        assert ho.ss_cross(bra, ket)[0, 0] == pytest.approx(ref, rel=1e-14, abs=1e-300)
        # the general Obara-Saika path reproduces the s closed form
        e = ho.eri_general(shells, bra, ket, [0], [0])[0, 0, 0, 0, 0]
        assert e == pytest.approx(ref, rel=1e-12, abs=1e-300)


def test_overlap_pins(golden):
    g = golden("integrals")
    for row in g["overlaps"]:
        a = ho.OShell(row[0:3], [tuple(row[6:8])])
        b = ho.OShell(row[3:6], [tuple(row[8:10]), tuple(row[10:12])])
        assert ho.overlap_s(a, b) == pytest.approx(row[12], rel=1e-14)


def test_generator_and_hilbert_match_reference(golden):
    g = golden("integrals")
    for k in range(3):
        s = inputs.generate_cluster(int(g[f"geo{k}_n"]), seed=int(g[f"geo{k}_seed"]))
        assert np.array_equal(np.array([sh.center for sh in s.shells]), g[f"geo{k}_centers"])
        _, perm = inputs.hilbert_order(s)
        assert np.array_equal(perm, g[f"geo{k}_perm"])


def test_product_weights_match_oracle():
    for l in (0, 1):
        prims = [(1.5, 0.5), (0.4, 0.5)]
        sh = basis.GaussianShell(center=[0.1, 0.2, 0.3], primitives=prims, l=l)
        o = ho.OShell(sh.center, prims, l=l)
        assert np.allclose(sh.weights, o.weights, rtol=1e-15, atol=0)


def test_case_label_table_matches():
    assert ho.CASE_LABELS == CASES


def test_splitmix_block_matches_sequential():
    rng = inputs.SplitMix64(12345)
    seq = [rng.next_u64() for _ in range(50)]
    blk = configs.splitmix64_block(12345, 0, 50)
    assert [int(x) for x in blk] == seq
    blk2 = configs.splitmix64_block(12345, 10, 5)
    assert [int(x) for x in blk2] == seq[10:15]
