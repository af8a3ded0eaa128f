"""Pin the oracle's p-shell extension (parity unpinned by the s-only reference).

Checks (SURVEY.md 8c "not pinned" item 1):
  - derivative identity p_x(A) = (1/2a) d/dA_x s(A), Richardson-extrapolated
    central differences, for every class reachable by one derivative;
  - 8-fold permutational symmetry, Cauchy-Schwarz, rotational covariance;
  - drivers: naive == symmetric == dense, and the direct-SCF set identity.
"""

import itertools

import numpy as np
import pytest

from oracle import hexfock_oracle as ho
from paper_1401_6961_b200 import basis, configs, inputs


def _shell(rng, l, center=None):
    k = int(rng.integers(1, 3))
    prims = list(zip(rng.uniform(0.2, 4.0, k), rng.uniform(0.3, 1.0, k)))
    c = rng.normal(scale=1.2, size=3) if center is None else center
    return ho.OShell(c, prims, l=l)


def _block(shells):
    bra = ho.Pairs(shells, [(0, 1)])
    ket = ho.Pairs(shells, [(2, 3)])
    return ho.eri_general(shells, bra, ket, [0], [0])[0]


def _lowered(sh):
    """s shell whose A-derivative is sh's p shell: weights w_p / (2a)."""
    s = ho.OShell(sh.center.copy(), list(zip(sh.exponents, sh.coefs)), l=0)
    s.weights = sh.weights / (2.0 * sh.exponents)
    return s


def _moved(sh, axis, h):
    m = ho.OShell(sh.center.copy(), list(zip(sh.exponents, sh.coefs)), l=sh.l)
    m.weights = sh.weights.copy()
    m.center = sh.center.copy()
    m.center[axis] += h
    return m


def _deriv(shells, pos, axis, h=2e-3):
    def f(step):
        s = list(shells)
        s[pos] = _moved(shells[pos], axis, step)
        return _block(s)

    d1 = (f(h) - f(-h)) / (2 * h)
    d2 = (f(h / 2) - f(-h / 2)) / h
    return (4 * d2 - d1) / 3


@pytest.mark.parametrize("cls", [c for c in itertools.product((0, 1), repeat=4) if any(c)])
def test_derivative_identity(cls):
    rng = np.random.default_rng(100 + sum(v << i for i, v in enumerate(cls)))
    shells = [_shell(rng, l) for l in cls]
    ref = _block(shells)
    pos = max(i for i in range(4) if cls[i])        # differentiate the last p
    low = list(shells)
    low[pos] = _lowered(shells[pos])
    scale = np.abs(ref).max()
    for axis in range(3):
        d = _deriv(low, pos, axis)
        idx = [slice(None)] * 4
        idx[pos] = axis
        got = ref[tuple(idx)]
        dd = d[tuple(slice(None) if i != pos else 0 for i in range(4))]
        assert np.abs(got - dd).max() <= 1e-8 * max(scale, 1e-3)


def test_permutational_symmetry_and_schwarz():
    rng = np.random.default_rng(7)
    for _ in range(8):
        ls = rng.integers(0, 2, size=4)
        sh = [_shell(rng, int(l)) for l in ls]
        e = _block(sh)
        assert np.allclose(_block([sh[1], sh[0], sh[2], sh[3]]), e.transpose(1, 0, 2, 3), rtol=1e-12, atol=1e-15)
        assert np.allclose(_block([sh[0], sh[1], sh[3], sh[2]]), e.transpose(0, 1, 3, 2), rtol=1e-12, atol=1e-15)
        assert np.allclose(_block([sh[2], sh[3], sh[0], sh[1]]), e.transpose(2, 3, 0, 1), rtol=1e-12, atol=1e-15)
        qb = _block([sh[0], sh[1], sh[0], sh[1]])
        qk = _block([sh[2], sh[3], sh[2], sh[3]])
        for a, b, c, d in itertools.product(*[range(n) for n in e.shape]):
            assert abs(e[a, b, c, d]) <= np.sqrt(qb[a, b, a, b] * qk[c, d, c, d]) * (1 + 1e-12) + 1e-300


def test_rotational_covariance():
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
    sh = [_shell(rng, l) for l in (1, 0, 1, 1)]
    e = _block(sh)
    rot = []
    for s in sh:
        r = ho.OShell(q @ s.center, list(zip(s.exponents, s.coefs)), l=s.l)
        rot.append(r)
    er = _block(rot)
    want = np.einsum("ai,ck,dl,ijkl->ajcd", q, q, q, e)
    assert np.allclose(er, want, rtol=1e-11, atol=1e-14)


def _small_p_system(units=2, seed=9):
    cfg = configs.cube_cluster(units, seed, "tiny")
    return cfg.system, cfg.P


def test_p_drivers_match_dense():
    system, P = _small_p_system(2)
    st = ho.Setup(system, P, tau_ovlp=0.0, leaf_size=4)
    K_dense = ho.dense_exchange(st.shells, P)
    K_n, cn = st.naive(0.0)
    K_s, cs = st.symmetric(0.0)
    assert np.abs(K_n - K_dense).max() <= 1e-12
    assert np.abs(K_s - K_dense).max() <= 1e-12
    ns = system.n_shells
    assert cn.eri_shell_quartets == ns ** 4
    assert cs.eri_shell_quartets == (ns * (ns + 1) // 2) ** 2


def test_p_direct_scf_set_identity():
    system, P = _small_p_system(3, seed=4)
    st = ho.Setup(system, P, tau_ovlp=0.0, leaf_size=6)
    log = []
    K_n, c = st.naive(1e-6, quartet_log=log)
    ref_log = []
    K_ref, skipped = ho.dense_exchange_screened(st.shells, P, 1e-6, quartet_log=ref_log)
    assert set(log) == set(ref_log)
    assert np.abs(K_n - K_ref).max() <= 1e-12
    K_s, _ = st.symmetric(1e-6)
    assert np.abs(K_s - K_n).max() <= 1e-12


def test_hilbert_order_keeps_l():
    system, _ = _small_p_system(2)
    s2, _ = inputs.hilbert_order(system)
    assert sorted(sh.l for sh in s2.shells) == sorted(sh.l for sh in system.shells)
    assert s2.n_functions == system.n_functions
