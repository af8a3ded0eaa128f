"""Device Hilbert reordering (csrc/prep.cu, hxf_hilbert_order)
against the host restatement of basis.py:275-331 (itself pinned to the reference's
golden permutations in test_oracle_golden.py) and those golden permutations.

CPU tests: argument errors (raised before any device work) and the loud no-device
failure.  GPU tests: bitwise-equal permutations and keys on clusters, the golden
geometries, ragged/degenerate inputs (zero extent on an axis, duplicate centres:
stability), bits 1 and 20, and a c5-sized system."""

import ctypes

import numpy as np
import pytest

from conftest import has_cuda, load_golden
from paper_1401_6961_b200 import _native, basis, inputs, prep, quadtree
from paper_1401_6961_b200.basis import InvalidArgumentError


def _host_keys(centers, bits):
    centers = np.asarray(centers, dtype=np.float64)
    lo = centers.min(axis=0)
    extent = centers.max(axis=0) - lo
    side = (1 << bits) - 1
    lattice = np.zeros_like(centers, dtype=np.int64)
    for ax in range(3):
        if extent[ax] > 0.0:
            lattice[:, ax] = np.rint((centers[:, ax] - lo[ax]) / extent[ax] * side)
    keys = inputs.hilbert_keys(lattice, bits).astype(np.uint64)
    perm = np.argsort(keys, kind="stable")
    return keys[perm], perm


@pytest.mark.parametrize("bits", [0, 21, -3])
def test_bad_bits_rejected(bits):
    s = inputs.generate_cluster(2, seed=1)
    with pytest.raises(InvalidArgumentError, match="bits_per_axis"):
        prep.hilbert_order_device(s, bits)
    with pytest.raises(InvalidArgumentError, match="bits_per_axis"):
        prep.hilbert_keys_and_perm(np.zeros((4, 3)), bits)


def test_c_abi_rejects_null_centers():
    rc = _native.lib().hxf_hilbert_order(None, ctypes.c_int64(3), 10, 0, None, None, None)
    assert rc == _native.HXF_EINVAL


@pytest.mark.skipif(has_cuda(), reason="checks the no-device path")
def test_no_device_fails_loudly():
    with pytest.raises(RuntimeError, match="no CUDA device"):
        prep.hilbert_keys_and_perm(np.zeros((4, 3)), 10)


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed", [(1, 3), (3, 3), (10, 5), (64, 11)])
def test_cluster_perm_matches_host(n, seed):
    s = inputs.generate_cluster(n, seed=seed)
    s_h, p_h = inputs.hilbert_order(s)
    s_d, p_d = prep.hilbert_order_device(s)
    assert np.array_equal(p_h, p_d)
    assert [sh.function_offset for sh in s_h.shells] == [sh.function_offset for sh in s_d.shells]
    assert np.array_equal(np.array([sh.center for sh in s_h.shells]),
                          np.array([sh.center for sh in s_d.shells]))


@pytest.mark.gpu
def test_golden_perms():
    g = load_golden("integrals")
    for k in range(3):
        s = inputs.generate_cluster(int(g[f"geo{k}_n"]), seed=int(g[f"geo{k}_seed"]))
        _, perm = prep.hilbert_order_device(s)
        assert np.array_equal(perm, g[f"geo{k}_perm"])


@pytest.mark.gpu
@pytest.mark.parametrize("bits", [1, 2, 7, 10, 16, 20])
def test_keys_bitwise_random(bits):
    rng = np.random.default_rng(bits)
    c = rng.uniform(-30.0, 30.0, size=(2000, 3))
    c[::7] = c[3]            # duplicate centres: stability of the sort
    c[::13, 1] = 0.5         # repeated coordinates on one axis
    k_d, p_d = prep.hilbert_keys_and_perm(c, bits)
    k_h, p_h = _host_keys(c, bits)
    assert np.array_equal(k_d, k_h)
    assert np.array_equal(p_d, p_h)


@pytest.mark.gpu
def test_degenerate_extents():
    line = np.zeros((50, 3))
    line[:, 2] = np.linspace(-4.0, 4.0, 50)[::-1]     # zero extent on x and y
    for c in (line, np.ones((5, 3)), np.zeros((1, 3))):
        k_d, p_d = prep.hilbert_keys_and_perm(c, 10)
        k_h, p_h = _host_keys(c, 10)
        assert np.array_equal(k_d, k_h) and np.array_equal(p_d, p_h)
    k, p = prep.hilbert_keys_and_perm(np.zeros((0, 3)), 10)
    assert k.size == 0 and p.size == 0


@pytest.mark.gpu
def test_half_way_lattice_rounding():
    """(c - lo) / extent * side landing on .5 exactly: rint is half-to-even on both sides."""
    side = (1 << 3) - 1
    xs = np.array([0.0, 0.5, 1.5, 2.5, 3.5, float(side)])   # extent = side: lattice = rint(x)
    c = np.stack([xs, xs[::-1], np.zeros_like(xs)], axis=1)
    k_d, p_d = prep.hilbert_keys_and_perm(c, 3)
    k_h, p_h = _host_keys(c, 3)
    assert np.array_equal(k_d, k_h) and np.array_equal(p_d, p_h)


@pytest.mark.gpu
def test_c5_sized_system():
    """BASELINE config 5's shell count (20480): the device permutation is the host's."""
    rng = np.random.default_rng(5)
    c = rng.normal(0.0, 25.0, size=(20480, 3))
    c[1::3] = c[0::3] + 1e-3   # close neighbours, like the H atoms of a water
    k_d, p_d = prep.hilbert_keys_and_perm(c, 10)
    k_h, p_h = _host_keys(c, 10)
    assert np.array_equal(p_d, p_h) and np.array_equal(k_d, k_h)
    assert np.all(np.diff(k_d.astype(np.int64)) >= 0)


# ---------------------------------------------------------------- partition build

def _tree(node):
    if node.is_leaf:
        return (node.shell_lo, node.shell_hi, node.fn_lo, node.fn_hi)
    return (node.shell_lo, node.shell_hi, node.fn_lo, node.fn_hi, _tree(node.left), _tree(node.right))


def _system_of_sizes(sizes):
    shells = [basis.GaussianShell(center=[0.1 * i, 0.0, 0.0], primitives=[(1.0, 1.0)], l=1 if s == 3 else 0)
              for i, s in enumerate(sizes)]
    return basis.BasisSystem(shells=basis.assign_offsets(shells), atoms=[])


def test_partition_leaf_size_below_largest_shell():
    with pytest.raises(InvalidArgumentError, match="leaf_size must be >= the largest shell"):
        prep.partition_levels_device([1, 3, 1], 2)
    with pytest.raises(InvalidArgumentError):
        prep.partition_levels_device([1, 0, 1], 4)


@pytest.mark.skipif(has_cuda(), reason="checks the no-device path")
def test_partition_no_device_fails_loudly():
    with pytest.raises(RuntimeError, match="no CUDA device"):
        prep.partition_levels_device([1, 1, 1], 2)


@pytest.mark.gpu
@pytest.mark.parametrize("leaf", [3, 4, 7, 10, 32])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_partition_ragged_matches_host(leaf, seed):
    rng = np.random.default_rng(seed)
    sizes = rng.choice([1, 3], size=int(rng.integers(1, 700)), p=[0.6, 0.4]).tolist()
    s = _system_of_sizes(sizes)
    host = quadtree.build_partition(s, leaf_size=leaf)
    dev = prep.build_partition_device(s, leaf_size=leaf)
    assert _tree(dev.root) == _tree(host.root)
    assert [[(x.shell_lo, x.shell_hi) for x in lv] for lv in dev.levels] == \
           [[(x.shell_lo, x.shell_hi) for x in lv] for lv in host.levels]


@pytest.mark.gpu
def test_partition_ties_and_small_cases():
    # midpoint exactly between two boundaries (ties go left), single shells, one leaf
    for sizes, leaf in (([1, 1], 1), ([1, 1, 1], 1), ([3, 1, 3], 3), ([1] * 10, 10), ([3], 3),
                        ([1, 3, 3, 1], 4), ([3] * 17, 3)):
        s = _system_of_sizes(sizes)
        assert _tree(prep.build_partition_device(s, leaf).root) == \
               _tree(quadtree.build_partition(s, leaf).root), (sizes, leaf)


@pytest.mark.gpu
def test_partition_cluster_and_c5_size():
    s, _ = inputs.hilbert_order(inputs.generate_cluster(40, seed=7))
    assert _tree(prep.build_partition_device(s).root) == _tree(quadtree.build_partition(s).root)
    sizes = [1, 1, 1, 3, 3] * 4096   # 20480 shells, 28672 functions (config 5's basis mix)
    s = _system_of_sizes(sizes)
    assert _tree(prep.build_partition_device(s, 10).root) == _tree(quadtree.build_partition(s, 10).root)
