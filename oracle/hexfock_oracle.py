"""CPU restatement of the reference's hierarchical exchange build.

TEST INFRASTRUCTURE ONLY -- see ``oracle/__init__.py``.  The product never
imports this module; it is the checker the CUDA path is compared against and
the CPU baseline ``bench.py`` times.

What it restates (all paths relative to /root/reference/pkg/src/hexfock):

* shell normalisation ............ basis.py:78-87
* Boys F0 (series / erf) ........ integrals.py:27-55
* primitive pair tables ......... integrals.py:115-154
* (ss|ss) ERIs .................. integrals.py:157-206, diagonal 219-222
* contracted s overlap .......... integrals.py:58-64, quadtree.py:272-281
* ragged bisection partition .... quadtree.py:90-113
* density quadtree .............. quadtree.py:198-235 (fsum norms 20-25)
* shell-pair quadtree ........... quadtree.py:284-337, leaf caches 358-395
* naive hextree driver .......... exchange_naive.py:68-240
* 4-fold symmetric driver ....... exchange_symmetry.py:135-409
* dense / direct-SCF oracles .... oracle.py:47-108

Parity pin.  For s shells the restatement performs the reference's floating
point operations in the reference's order (Boys series, prefactor, weight
multiply, primitive sums), and ``tests/test_oracle_golden.py`` checks it
against golden vectors written by the reference itself
(``tests/golden/make_golden.py``): identical culled quartet sets and counters,
bit-identical tree norms, K within 1e-13.

p shells (BASELINE configs 2-5) are an extension -- the reference is s-only
 -- so for them parity is *unpinned by the reference*.  The
extension is pinned instead by (tests/test_oracle_pshell.py):
  - the s-limit of the general recursion reproducing the s closed form;
  - the derivative identity  p_x(A) = (1/2a) d/dA_x s(A), checked by
    Richardson-extrapolated central differences of the s integrals;
  - the 8-fold permutational symmetry of the ERI and Cauchy-Schwarz;
  - rotational covariance of the p blocks.
Definitions used for p shells (documented in DESIGN.md):
  - p shells are Cartesian (x, y, z), primitive norm (2a/pi)^{3/4}(4a)^{1/2};
  - overlap pruning uses the s-proxy overlap of the shells' primitives;
  - Q_ij = max over function pairs of (i_f j_f|i_f j_f), canonical orientation;
  - the per-quartet |P| factor is max |P| over the nu x lambda function block.
General-l ERIs use the Obara-Saika vertical recursion onto [e0|f0] followed by
the Head-Gordon-Pople horizontal transfer, written as a memoised recursion.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np
from scipy.special import erf

TWO_PI_POW_2_5 = 2.0 * math.pi ** 2.5
F0_SWITCH = 12.0
F0_TERMS = 70
CASE_LABELS = ("A", "B", "C", "D", "E", "F1", "F2", "H", "SPARSE")


class InvalidArgumentError(ValueError):
    pass


class LogicError(RuntimeError):
    pass


# --------------------------------------------------------------------------
# basis (basis.py:62-87, extended to Cartesian p)

class OShell:
    """Oracle-side shell: center (Bohr), exponents, normalised weights, l."""

    __slots__ = ("center", "exponents", "coefs", "weights", "sweights", "l",
                 "nfn", "fn")

    def __init__(self, center, primitives, l=0, fn=0):
        self.center = np.asarray(center, dtype=float)
        self.exponents = np.asarray([e for e, _ in primitives], dtype=float)
        self.coefs = np.asarray([c for _, c in primitives], dtype=float)
        self.l = int(l)
        self.nfn = 1 if self.l == 0 else 3
        self.fn = int(fn)
        self.sweights = s_weights(self.exponents, self.coefs)
        self.weights = (self.sweights if self.l == 0
                        else p_weights(self.exponents, self.coefs))


def s_weights(exps, coefs):
    # basis.py:84-87: fold primitive norms and overall normalisation
    w = coefs * (2.0 * exps / np.pi) ** 0.75
    p = exps[:, None] + exps[None, :]
    s = np.sum(w[:, None] * w[None, :] * (np.pi / p) ** 1.5)
    return w / math.sqrt(s)


def p_weights(exps, coefs):
    # Cartesian p_x = x exp(-a r^2): primitive norm (2a/pi)^{3/4} (4a)^{1/2};
    # <p_x|p_x> over a primitive pair = (pi/p)^{3/2} / (2p)
    w = coefs * (2.0 * exps / np.pi) ** 0.75 * np.sqrt(4.0 * exps)
    p = exps[:, None] + exps[None, :]
    s = np.sum(w[:, None] * w[None, :] * (np.pi / p) ** 1.5 / (2.0 * p))
    return w / math.sqrt(s)


def as_oracle_shells(system):
    """Duck-typed conversion: any shell with center/primitives (+ optional l)."""
    out = []
    off = 0
    for sh in system.shells:
        l = int(getattr(sh, "l", 0))
        o = OShell(sh.center, sh.primitives, l=l, fn=off)
        out.append(o)
        off += o.nfn
    return out


# --------------------------------------------------------------------------
# Boys function (integrals.py:27-55) and F_m for m <= 4

def boys_f0(t):
    t = np.asarray(t, dtype=float)
    if np.any(t < 0.0):
        raise InvalidArgumentError("boys_f0 requires t >= 0")
    scalar = t.ndim == 0
    t = np.atleast_1d(t)
    out = np.empty_like(t)
    lo = t < F0_SWITCH
    if lo.any():
        ts = t[lo]
        two_t = 2.0 * ts
        term = np.ones_like(ts)
        acc = np.ones_like(ts)
        for k in range(1, F0_TERMS):
            term = term * two_t / (2 * k + 1)
            acc += term
        out[lo] = np.exp(-ts) * acc
    if (~lo).any():
        tl = t[~lo]
        st = np.sqrt(tl)
        out[~lo] = 0.5 * np.sqrt(np.pi) * erf(st) / st
    return float(out[0]) if scalar else out


def boys_fm(t, mmax):
    """[F_0..F_mmax](t), shape (mmax+1,) + t.shape.

    Below the switch: series for F_mmax then downward recursion; above it:
    erf form for F_0 then upward recursion (both stable in their range).
    """
    t = np.asarray(t, dtype=float)
    out = np.empty((mmax + 1,) + t.shape)
    et = np.exp(-t)
    lo = t < F0_SWITCH
    if lo.any():
        ts = t[lo]
        two_t = 2.0 * ts
        term = np.full_like(ts, 1.0 / (2 * mmax + 1))
        acc = term.copy()
        for k in range(1, F0_TERMS + 10):
            term = term * two_t / (2 * mmax + 2 * k + 1)
            acc += term
        f = et[lo] * acc
        out[mmax][lo] = f
        for m in range(mmax - 1, -1, -1):
            f = (two_t * f + et[lo]) / (2 * m + 1)
            out[m][lo] = f
    hi = ~lo
    if hi.any():
        tl = t[hi]
        st = np.sqrt(tl)
        f = 0.5 * np.sqrt(np.pi) * erf(st) / st
        out[0][hi] = f
        for m in range(mmax):
            f = ((2 * m + 1) * f - et[hi]) / (2.0 * tl)
            out[m + 1][hi] = f
    return out


# --------------------------------------------------------------------------
# primitive pair tables (integrals.py:115-154)

class Pairs:
    """Flattened primitive pair table over an ordered list of shell pairs."""

    def __init__(self, shells, pair_list):
        self.i = np.asarray([a for a, _ in pair_list], dtype=np.intp)
        self.j = np.asarray([b for _, b in pair_list], dtype=np.intp)
        offs = [0]
        ps, cs, ws, als = [], [], [], []
        for a, b in pair_list:
            A, B = shells[a], shells[b]
            ea, eb = A.exponents[:, None], B.exponents[None, :]
            p = (ea + eb).ravel()
            ab = (ea * eb).ravel()
            d = A.center - B.center
            r2 = float(np.dot(d, d))
            w = (A.weights[:, None] * B.weights[None, :]).ravel() * np.exp(-ab / p * r2)
            c = (ea[..., None] * A.center + eb[..., None] * B.center).reshape(-1, 3)
            c /= p[:, None]
            offs.append(offs[-1] + len(p))
            ps.append(p)
            cs.append(c)
            ws.append(w)
            als.append(np.broadcast_to(ea, (len(A.exponents), len(B.exponents))).ravel())
        self.off = np.asarray(offs, dtype=np.intp)
        self.p = np.concatenate(ps) if ps else np.empty(0)
        self.c = np.concatenate(cs) if cs else np.empty((0, 3))
        self.w = np.concatenate(ws) if ws else np.empty(0)
        self.alpha = np.concatenate(als) if als else np.empty(0)

    @property
    def n(self):
        return len(self.i)


# --------------------------------------------------------------------------
# (ss|ss) ERIs (integrals.py:157-206), same operation order as the reference

def ss_cross(bra, ket):
    if bra.n == 0 or ket.n == 0:
        return np.zeros((bra.n, ket.n))
    pq = bra.p[:, None] * ket.p[None, :]
    ps = bra.p[:, None] + ket.p[None, :]
    d = bra.c[:, None, :] - ket.c[None, :, :]
    r2 = np.einsum("ijk,ijk->ij", d, d)
    f0 = boys_f0((pq / ps * r2).ravel()).reshape(pq.shape)
    m = TWO_PI_POW_2_5 / (pq * np.sqrt(ps)) * bra.w[:, None] * ket.w[None, :] * f0
    m = np.add.reduceat(m, bra.off[:-1], axis=0)
    return np.add.reduceat(m, ket.off[:-1], axis=1)


def ss_elementwise(bra, ket, ia, ib):
    ia = np.asarray(ia, dtype=np.intp)
    ib = np.asarray(ib, dtype=np.intp)
    out = np.zeros(len(ia))
    na = bra.off[ia + 1] - bra.off[ia]
    nb = ket.off[ib + 1] - ket.off[ib]
    for ca in np.unique(na):
        for cb in np.unique(nb):
            sel = np.nonzero((na == ca) & (nb == cb))[0]
            if len(sel) == 0:
                continue
            ga = bra.off[ia[sel], None] + np.arange(ca)[None, :]
            gb = ket.off[ib[sel], None] + np.arange(cb)[None, :]
            p1, w1, c1 = bra.p[ga], bra.w[ga], bra.c[ga]
            p2, w2, c2 = ket.p[gb], ket.w[gb], ket.c[gb]
            pq = p1[:, :, None] * p2[:, None, :]
            ps = p1[:, :, None] + p2[:, None, :]
            d = c1[:, :, None, :] - c2[:, None, :, :]
            r2 = np.einsum("nijk,nijk->nij", d, d)
            f0 = boys_f0((pq / ps * r2).ravel()).reshape(pq.shape)
            v = TWO_PI_POW_2_5 / (pq * np.sqrt(ps)) * f0
            v *= w1[:, :, None] * w2[:, None, :]
            out[sel] = v.sum(axis=(1, 2))
    return out


# --------------------------------------------------------------------------
# general l <= 1 ERIs: Obara-Saika VRR onto [e0|f0], contraction, HGP HRR

_UNIT = ((1, 0, 0), (0, 1, 0), (0, 0, 1))


def _cart(l):
    return [(0, 0, 0)] if l == 0 else list(_UNIT)


def _sub(v, i):
    return v[:i] + (v[i] - 1,) + v[i + 1:]


def _add(v, i):
    return v[:i] + (v[i] + 1,) + v[i + 1:]


def _carts_upto(lo, hi):
    out = []
    for L in range(lo, hi + 1):
        for x in range(L, -1, -1):
            for y in range(L - x, -1, -1):
                out.append((x, y, L - x - y))
    return out


def eri_general(shells, bra, ket, ia, ib):
    """Contracted Cartesian blocks (ij|kl) for quartets of one angular class.

    All quartets (bra pair ia[n], ket pair ib[n]) must share (li,lj,lk,ll)
    and primitive counts; returns (n, ni, nj, nk, nl).
    """
    ia = np.asarray(ia, dtype=np.intp)
    ib = np.asarray(ib, dtype=np.intp)
    n = len(ia)
    si, sj = shells[bra.i[ia[0]]], shells[bra.j[ia[0]]]
    sk, sl = shells[ket.i[ib[0]]], shells[ket.j[ib[0]]]
    la, lb, lc, ld = si.l, sj.l, sk.l, sl.l
    L = la + lb + lc + ld
    ka = bra.off[ia[0] + 1] - bra.off[ia[0]]
    kb = ket.off[ib[0] + 1] - ket.off[ib[0]]
    ga = bra.off[ia, None] + np.arange(ka)[None, :]          # (n, ka)
    gb = ket.off[ib, None] + np.arange(kb)[None, :]          # (n, kb)
    p = bra.p[ga][:, :, None]                               # (n, ka, 1)
    q = ket.p[gb][:, None, :]                               # (n, 1, kb)
    P = bra.c[ga][:, :, None, :]                            # (n, ka, 1, 3)
    Q = ket.c[gb][:, None, :, :]                            # (n, 1, kb, 3)
    A = np.stack([shells[t].center for t in bra.i[ia]])[:, None, None, :]
    B = np.stack([shells[t].center for t in bra.j[ia]])[:, None, None, :]
    C = np.stack([shells[t].center for t in ket.i[ib]])[:, None, None, :]
    D = np.stack([shells[t].center for t in ket.j[ib]])[:, None, None, :]
    pq = p * q
    ps = p + q
    rho = pq / ps
    W = (p[..., None] * P + q[..., None] * Q) / ps[..., None]
    d = P - Q
    T = rho * np.einsum("nabk,nabk->nab", d, d)
    Fm = boys_fm(T, L)
    pref = TWO_PI_POW_2_5 / (pq * np.sqrt(ps)) * bra.w[ga][:, :, None] * ket.w[gb][:, None, :]
    PA = np.broadcast_to(P - A, W.shape)
    WP = W - P
    QC = np.broadcast_to(Q - C, W.shape)
    WQ = W - Q
    memo = {}
    zero = (0, 0, 0)

    def vrr(e, f, m):
        key = (e, f, m)
        hit = memo.get(key)
        if hit is not None:
            return hit
        if e == zero and f == zero:
            v = pref * Fm[m]
        elif e != zero:
            i = next(t for t in range(3) if e[t] > 0)
            e1 = _sub(e, i)
            v = PA[..., i] * vrr(e1, f, m) + WP[..., i] * vrr(e1, f, m + 1)
            if e1[i] > 0:
                e2 = _sub(e1, i)
                v = v + e1[i] / (2.0 * p) * (vrr(e2, f, m) - rho / p * vrr(e2, f, m + 1))
            if f[i] > 0:
                v = v + f[i] / (2.0 * ps) * vrr(e1, _sub(f, i), m + 1)
        else:
            i = next(t for t in range(3) if f[t] > 0)
            f1 = _sub(f, i)
            v = QC[..., i] * vrr(e, f1, m) + WQ[..., i] * vrr(e, f1, m + 1)
            if f1[i] > 0:
                f2 = _sub(f1, i)
                v = v + f1[i] / (2.0 * q) * (vrr(e, f2, m) - rho / q * vrr(e, f2, m + 1))
        memo[key] = v
        return v

    # contracted [e0|f0] over the primitive axes
    E = {}
    for e in _carts_upto(la, la + lb):
        for f in _carts_upto(lc, lc + ld):
            E[(e, f)] = vrr(e, f, 0).sum(axis=(1, 2))
    AB = (A - B)[:, 0, 0, :]
    CD = (C - D)[:, 0, 0, :]
    memo_h = {}

    def hrr(a, b, c, dd):
        key = (a, b, c, dd)
        hit = memo_h.get(key)
        if hit is not None:
            return hit
        if b != zero:
            i = next(t for t in range(3) if b[t] > 0)
            b1 = _sub(b, i)
            v = hrr(_add(a, i), b1, c, dd) + AB[:, i] * hrr(a, b1, c, dd)
        elif dd != zero:
            i = next(t for t in range(3) if dd[t] > 0)
            d1 = _sub(dd, i)
            v = hrr(a, b, _add(c, i), d1) + CD[:, i] * hrr(a, b, c, d1)
        else:
            v = E[(a, c)]
        memo_h[key] = v
        return v

    ca, cb, cc, cd = _cart(la), _cart(lb), _cart(lc), _cart(ld)
    out = np.empty((n, len(ca), len(cb), len(cc), len(cd)))
    for x, a in enumerate(ca):
        for y, b in enumerate(cb):
            for z, c in enumerate(cc):
                for t, dd in enumerate(cd):
                    out[:, x, y, z, t] = hrr(a, b, c, dd)
    return out


def eri_blocks(shells, bra, ket, ia, ib):
    """Blocks for arbitrary quartets, grouped internally by class/primitives.

    Returns a list of (n_i, n_j, n_k, n_l) arrays aligned with (ia, ib).  All-s
    quartets go through the reference-ordered closed form.
    """
    ia = np.asarray(ia, dtype=np.intp)
    ib = np.asarray(ib, dtype=np.intp)
    out = [None] * len(ia)
    if len(ia) == 0:
        return out
    lv = np.asarray([sh.l for sh in shells])
    key_b = lv[bra.i[ia]] * 2 + lv[bra.j[ia]]
    key_k = lv[ket.i[ib]] * 2 + lv[ket.j[ib]]
    cls = key_b * 4 + key_k
    na = bra.off[ia + 1] - bra.off[ia]
    nb = ket.off[ib + 1] - ket.off[ib]
    s_sel = np.nonzero(cls == 0)[0]
    if len(s_sel):
        v = ss_elementwise(bra, ket, ia[s_sel], ib[s_sel])
        for t, x in zip(s_sel, v):
            out[t] = np.full((1, 1, 1, 1), x)
    rest = np.nonzero(cls != 0)[0]
    if len(rest):
        keys = np.stack([cls[rest], na[rest], nb[rest]], axis=1)
        uniq, inv = np.unique(keys, axis=0, return_inverse=True)
        inv = inv.ravel()
        for g in range(len(uniq)):
            sel = rest[inv == g]
            blk = eri_general(shells, bra, ket, ia[sel], ib[sel])
            for t, x in zip(sel, blk):
                out[t] = x
    return out


def diagonal_q(shells, pairs):
    """Q per pair = max_f (i_f j_f|i_f j_f) (for s: integrals.py:219-222)."""
    idx = np.arange(pairs.n)
    lv = np.asarray([sh.l for sh in shells])
    if pairs.n and not np.any(lv[pairs.i]) and not np.any(lv[pairs.j]):
        return ss_elementwise(pairs, pairs, idx, idx)
    blocks = eri_blocks(shells, pairs, pairs, idx, idx)
    q = np.empty(pairs.n)
    for t, blk in enumerate(blocks):
        ni, nj = blk.shape[0], blk.shape[1]
        q[t] = max(blk[x, y, x, y] for x in range(ni) for y in range(nj))
    return q


# --------------------------------------------------------------------------
# overlap (integrals.py:58-64), s-proxy for p shells

def overlap_s(a, b):
    d = a.center - b.center
    r2 = float(np.dot(d, d))
    ea, eb = a.exponents[:, None], b.exponents[None, :]
    p = ea + eb
    s = (np.pi / p) ** 1.5 * np.exp(-ea * eb / p * r2)
    return float(np.sum(a.sweights[:, None] * b.sweights[None, :] * s))


def overlap_matrix(shells):
    n = len(shells)
    s = np.zeros((n, n))
    for i in range(n):
        for j in range(i, n):
            v = overlap_s(shells[i], shells[j])
            s[i, j] = v
            s[j, i] = v
    return s


# --------------------------------------------------------------------------
# partition (quadtree.py:28-113)

class OSpan:
    __slots__ = ("slo", "shi", "flo", "fhi", "left", "right")

    def __init__(self, slo, shi, flo, fhi):
        self.slo, self.shi, self.flo, self.fhi = slo, shi, flo, fhi
        self.left = self.right = None

    @property
    def is_leaf(self):
        return self.left is None

    def kids(self):
        return (self,) if self.left is None else (self.left, self.right)


def build_partition(sizes, leaf_size=10):
    sizes = list(sizes)
    if leaf_size < max(sizes, default=1):
        raise InvalidArgumentError("leaf_size must be >= the largest shell")
    cum = np.concatenate([[0], np.cumsum(sizes)]).astype(int)

    def split(lo, hi):
        s = OSpan(lo, hi, int(cum[lo]), int(cum[hi]))
        if s.fhi - s.flo <= leaf_size:
            return s
        mid = (s.flo + s.fhi) / 2.0
        cand = np.arange(lo + 1, hi)
        b = int(cand[int(np.argmin(np.abs(cum[cand] - mid)))])  # first = left tie
        s.left = split(lo, b)
        s.right = split(b, hi)
        return s

    return split(0, len(sizes))


# --------------------------------------------------------------------------
# density quadtree (quadtree.py:198-235)

def _rss(vals):
    return math.sqrt(math.fsum(v * v for v in vals))


class MNode:
    __slots__ = ("row", "col", "norm", "children", "leaf")

    def __init__(self, row, col, norm, children=None, leaf=None):
        self.row, self.col, self.norm = row, col, norm
        self.children = children or {}
        self.leaf = leaf

    def child(self, a, b):
        if self.leaf is not None:
            return self if (a, b) == (0, 0) else None
        return self.children.get((a, b))


def build_matrix_tree(P, root, zero_drop=0.0):
    P = np.asarray(P, dtype=float)

    def build(r, c):
        if r.is_leaf and c.is_leaf:
            blk = P[r.flo:r.fhi, c.flo:c.fhi]
            if not np.any(blk):
                return None
            nrm = math.sqrt(math.fsum((blk ** 2).ravel().tolist()))
            if nrm <= zero_drop:
                return None
            return MNode(r, c, nrm, leaf=blk)
        kids = {}
        for a, rr in enumerate(r.kids()):
            for b, cc in enumerate(c.kids()):
                ch = build(rr, cc)
                if ch is not None:
                    kids[(a, b)] = ch
        if not kids:
            return None
        return MNode(r, c, _rss(ch.norm for ch in kids.values()), children=kids)

    t = build(root, root)
    if t is None:
        t = MNode(root, root, 0.0, leaf=P if root.is_leaf else None)
    return t


# --------------------------------------------------------------------------
# shell-pair quadtree (quadtree.py:238-337) and leaf caches (:358-395)

class PNode:
    __slots__ = ("row", "col", "pruned", "children", "diag", "diag_norm",
                 "rowsum_max", "colsum_max", "pairs", "cache")

    def __init__(self, row, col):
        self.row, self.col = row, col
        self.pruned = False
        self.children = {}
        self.diag = None
        self.diag_norm = self.rowsum_max = self.colsum_max = 0.0
        self.pairs = None
        self.cache = {}

    @property
    def is_leaf(self):
        return self.row.is_leaf and self.col.is_leaf

    def child(self, a, b):
        if self.is_leaf:
            return self if (a, b) == (0, 0) else None
        return self.children.get((a, b))


def build_pair_tree(shells, root, tau_ovlp=0.0, s_abs=None):
    if s_abs is None:
        s_abs = np.abs(overlap_matrix(shells))

    def build(r, c):
        nd = PNode(r, c)
        if s_abs[r.slo:r.shi, c.slo:c.shi].max() < tau_ovlp:
            nd.pruned = True
            return nd
        if nd.is_leaf:
            plist = [(i, j) for i in range(r.slo, r.shi) for j in range(c.slo, c.shi)]
            nd.pairs = Pairs(shells, plist)
            canon = Pairs(shells, [(min(i, j), max(i, j)) for i, j in plist])
            q = diagonal_q(shells, canon).reshape(r.shi - r.slo, c.shi - c.slo)
            nd.diag = q
            nd.diag_norm = math.sqrt(math.fsum((q ** 2).ravel().tolist()))
            nd.rowsum_max = float(q.sum(axis=1).max())
            nd.colsum_max = float(q.sum(axis=0).max())
            return nd
        rk, ck = r.kids(), c.kids()
        for a in range(len(rk)):
            for b in range(len(ck)):
                nd.children[(a, b)] = build(rk[a], ck[b])
        live = [ch for ch in nd.children.values() if not ch.pruned]
        if not live:
            nd.pruned = True
            nd.children = {}
            return nd
        nd.diag_norm = _rss(ch.diag_norm for ch in live)
        nd.rowsum_max = max(math.fsum(nd.children[(a, b)].rowsum_max for b in range(len(ck)))
                            for a in range(len(rk)))
        nd.colsum_max = max(math.fsum(nd.children[(a, b)].colsum_max for a in range(len(rk)))
                            for b in range(len(ck)))
        return nd

    return build(root, root)


def _subset(pd, idx, shells):
    sub = Pairs.__new__(Pairs)
    idx = np.asarray(idx, dtype=np.intp)
    lens = pd.off[idx + 1] - pd.off[idx]
    sub.off = np.concatenate([[0], np.cumsum(lens)]).astype(np.intp)
    g = (np.concatenate([np.arange(pd.off[t], pd.off[t + 1]) for t in idx])
         if len(idx) else np.empty(0, dtype=np.intp))
    sub.i, sub.j = pd.i[idx], pd.j[idx]
    sub.p, sub.c, sub.w, sub.alpha = pd.p[g], pd.c[g], pd.w[g], pd.alpha[g]
    return sub


def leaf_cache(node, shells, canonical=False):
    key = "canon" if canonical else "full"
    hit = node.cache.get(key)
    if hit is not None:
        return hit
    pd = node.pairs
    q = node.diag.ravel()
    if canonical and node.row is node.col:
        ns = node.row.shi - node.row.slo
        keep = np.asarray([x * ns + y for x in range(ns) for y in range(x, ns)], dtype=np.intp)
        pd = _subset(pd, keep, shells)
        q = q[keep]
    fn = np.asarray([sh.fn for sh in shells])
    nf = np.asarray([sh.nfn for sh in shells])
    c = {"pd": pd, "q": q, "fi": fn[pd.i], "fj": fn[pd.j], "ni": nf[pd.i], "nj": nf[pd.j],
         "wd": (pd.i != pd.j).astype(float)}
    node.cache[key] = c
    return c


# --------------------------------------------------------------------------
# drivers (exchange_naive.py, exchange_symmetry.py)

class Counters:
    FIELDS = ("tasks_visited", "tasks_culled_screening", "tasks_culled_absent",
              "leaf_contractions", "eri_shell_quartets", "quartets_culled_leaf",
              "tasks_expanded", "children_spawned")

    def __init__(self, symmetric=False):
        for f in self.FIELDS:
            setattr(self, f, 0)
        self.culled_bound_ledger = 0.0
        self.symmetric = symmetric
        if symmetric:
            self.links_culled_screening = 0
            self.links_culled_absent = 0
            self.case_tasks = {c: 0 for c in CASE_LABELS}
            self.case_leaf_tasks = {c: 0 for c in CASE_LABELS}

    def merge(self, o):
        for f in self.FIELDS:
            setattr(self, f, getattr(self, f) + getattr(o, f))
        self.culled_bound_ledger += o.culled_bound_ledger
        if self.symmetric:
            self.links_culled_screening += o.links_culled_screening
            self.links_culled_absent += o.links_culled_absent
            for c in CASE_LABELS:
                self.case_tasks[c] += o.case_tasks[c]
                self.case_leaf_tasks[c] += o.case_leaf_tasks[c]

    def to_dict(self):
        d = {f: getattr(self, f) for f in self.FIELDS}
        if self.symmetric:
            d["links_culled_screening"] = self.links_culled_screening
            d["links_culled_absent"] = self.links_culled_absent
        d["culled_bound_ledger"] = self.culled_bound_ledger
        if self.symmetric:
            d["case_tasks"] = dict(self.case_tasks)
            d["case_leaf_tasks"] = dict(self.case_leaf_tasks)
        return d


def sorted_product(a, b, c):
    lo, mid, hi = sorted((a, b, c))
    return lo * mid * hi


def culled_task_bound(b, pn, k, tb=False, tk=False):
    bs = b.colsum_max if tb else b.rowsum_max
    ks = k.rowsum_max if tk else k.colsum_max
    return 0.5 * pn * math.sqrt(max(bs, 0.0)) * math.sqrt(max(ks, 0.0))


def _pmax_block(P, fj, nj, fk, nk):
    """|P| factor per (bra pair, ket pair): max |P| over the nu x lambda block."""
    if np.all(nj == 1) and np.all(nk == 1):
        return np.abs(P[np.ix_(fj, fk)])
    out = np.empty((len(fj), len(fk)))
    for a in range(len(fj)):
        for b in range(len(fk)):
            out[a, b] = np.abs(P[fj[a]:fj[a] + nj[a], fk[b]:fk[b] + nk[b]]).max()
    return out


def _accumulate(K, P, blocks, sel_a, sel_b, A, B, src, dst, weight):
    """K[dst] += -1/2 sum P[src] (ij|kl) for the given (bra, ket) pairs.

    src/dst name the function index pairs: 'jk'/'il' for slot 0, etc.
    """
    for t, (a, b) in enumerate(zip(sel_a, sel_b)):
        e = blocks[t]
        w = weight[t] if weight is not None else 1.0
        if w == 0.0:
            continue
        f = {"i": (A["fi"][a], A["ni"][a]), "j": (A["fj"][a], A["nj"][a]),
             "k": (B["fi"][b], B["ni"][b]), "l": (B["fj"][b], B["nj"][b])}
        (s0, sn0), (s1, sn1) = f[src[0]], f[src[1]]
        (d0, dn0), (d1, dn1) = f[dst[0]], f[dst[1]]
        pb = P[s0:s0 + sn0, s1:s1 + sn1]
        spec = "ijkl," + src + "->" + dst
        K[d0:d0 + dn0, d1:d1 + dn1] += w * (-0.5 * np.einsum(spec, e, pb))


class _Naive:
    def __init__(self, shells, P, n, tau, mode, evaluate, want_log):
        self.shells, self.P = shells, P
        self.K = np.zeros((n, n))
        self.c = Counters()
        self.tau, self.mode, self.evaluate = tau, mode, evaluate
        self.qlog = [] if want_log else None
        self.spawn = None

    def visit(self, b, p, k, depth=1):
        c = self.c
        c.tasks_visited += 1
        if b is None or p is None or k is None or b.pruned or k.pruned:
            c.tasks_culled_absent += 1
            return
        fb, fk = b.diag_norm, k.diag_norm
        if self.mode == "schwarz":
            fb, fk = math.sqrt(fb), math.sqrt(fk)
        if sorted_product(fb, p.norm, fk) <= self.tau:
            c.tasks_culled_screening += 1
            c.culled_bound_ledger += culled_task_bound(b, p.norm, k)
            return
        if b.is_leaf and k.is_leaf:
            c.leaf_contractions += 1
            self.contract(b, p, k)
            return
        c.tasks_expanded += 1
        for a in range(len(b.row.kids())):
            for cc in range(len(b.col.kids())):
                bch = b.child(a, cc)
                for d in range(len(k.row.kids())):
                    pch = p.child(cc, d)
                    for bb in range(len(k.col.kids())):
                        c.children_spawned += 1
                        if self.spawn is not None and depth == 0:
                            self.spawn.append((bch, pch, k.child(d, bb)))
                        else:
                            self.visit(bch, pch, k.child(d, bb), depth + 1)

    def contract(self, b, p, k):
        c = self.c
        A, B = leaf_cache(b, self.shells), leaf_cache(k, self.shells)
        ma, mb = A["pd"].n, B["pd"].n
        sq_a, sq_b = np.sqrt(A["q"]), np.sqrt(B["q"])
        fa, fk = (sq_a, sq_b) if self.mode == "schwarz" else (A["q"], B["q"])
        pg = _pmax_block(self.P, A["fj"], A["nj"], B["fi"], B["ni"])
        bound = (fa[:, None] * pg) * fk[None, :]
        keep = bound > self.tau
        nkeep = int(keep.sum())
        c.eri_shell_quartets += nkeep
        if nkeep < ma * mb:
            c.quartets_culled_leaf += ma * mb - nkeep
            sb = bound if self.mode == "schwarz" else (sq_a[:, None] * pg) * sq_b[None, :]
            c.culled_bound_ledger += 0.5 * float(sb[~keep].sum())
        if not self.evaluate or nkeep == 0:
            return
        ia, ib = np.nonzero(keep)
        blocks = eri_blocks(self.shells, A["pd"], B["pd"], ia, ib)
        _accumulate(self.K, self.P, blocks, ia, ib, A, B, "jk", "il", None)
        if self.qlog is not None:
            self.qlog.extend(zip(A["pd"].i[ia].tolist(), A["pd"].j[ia].tolist(),
                                 B["pd"].i[ib].tolist(), B["pd"].j[ib].tolist()))


def exchange_naive(shells, bra, ket, Ptree, P, tau=0.0, mode="schwarz",
                   quartet_log=None, evaluate=True, threads=1):
    """exchange_naive.py:200-240 restated (function-level for p shells)."""
    if tau < 0.0:
        raise InvalidArgumentError("tau_2e must be non-negative")
    if mode not in ("schwarz", "literal"):
        raise InvalidArgumentError(f"unknown screening mode {mode!r}")
    n = bra.row.fhi
    want = quartet_log is not None
    run = _Naive(shells, P, n, tau, mode, evaluate, want)
    if threads > 1:
        run.spawn = []
        run.visit(bra, Ptree, ket, depth=0)

        def work(args):
            sub = _Naive(shells, P, n, tau, mode, evaluate, want)
            sub.visit(*args)
            return sub

        with ThreadPoolExecutor(max_workers=threads) as pool:
            subs = list(pool.map(work, run.spawn))
        for sub in subs:
            run.K += sub.K
            run.c.merge(sub.c)
            if want:
                run.qlog.extend(sub.qlog)
    else:
        run.visit(bra, Ptree, ket)
    if want:
        quartet_log.extend(run.qlog)
    return run.K, run.c


_SLOT_T = ((False, False), (True, False), (False, True), (True, True))


def case_label(b, k):
    """exchange_symmetry.py:135-173."""
    mu, nu, lam, sig = b.row, b.col, k.row, k.col
    if b is k:
        return "E"
    bd, kd = mu is nu, lam is sig
    if bd and kd:
        return "H"
    if bd or kd:
        return "B"
    if nu is lam or mu is sig:
        return "A"
    if mu is lam:
        return "F1"
    if nu is sig:
        return "F2"
    if nu.flo < lam.flo or sig.flo < mu.flo:
        return "A"
    if (lam.flo < mu.flo) != (sig.flo < nu.flo):
        return "C"
    return "D"


def _canon_keys(node):
    nr, nc = len(node.row.kids()), len(node.col.kids())
    if node.row is node.col:
        return [(a, b) for a in range(nr) for b in range(a, nc)]
    return [(a, b) for a in range(nr) for b in range(nc)]


class _Sym:
    def __init__(self, shells, P, n, tau, mode, evaluate, want_log):
        self.shells, self.P = shells, P
        self.K = np.zeros((n, n))
        self.c = Counters(symmetric=True)
        self.tau, self.mode, self.evaluate = tau, mode, evaluate
        self.qlog = [] if want_log else None
        self.spawn = None

    def visit(self, b, k, refs, alive, depth=1):
        c = self.c
        c.tasks_visited += 1
        if b.pruned or k.pruned:
            c.tasks_culled_absent += 1
            return
        fb, fk = b.diag_norm, k.diag_norm
        if self.mode == "schwarz":
            fb, fk = math.sqrt(fb), math.sqrt(fk)
        live = [False] * 4
        screened = absent = False
        for g in range(4):
            if not alive[g]:
                continue
            ref = refs[g]
            if ref is None:
                c.links_culled_absent += 1
                absent = True
                continue
            if sorted_product(fb, ref.norm, fk) <= self.tau:
                c.links_culled_screening += 1
                screened = True
                tb, tk = _SLOT_T[g]
                c.culled_bound_ledger += culled_task_bound(b, ref.norm, k, tb, tk)
                continue
            live[g] = True
        if not any(live):
            if screened:
                c.tasks_culled_screening += 1
            else:
                c.tasks_culled_absent += 1
            return
        label = "SPARSE" if absent else case_label(b, k)
        c.case_tasks[label] += 1
        if b.is_leaf and k.is_leaf:
            c.case_leaf_tasks[label] += 1
            c.leaf_contractions += 1
            self.contract(b, k, refs, live)
            return
        c.tasks_expanded += 1
        pnl, pml, pns, pms = refs
        kk = _canon_keys(k)
        for a, cc in _canon_keys(b):
            bch = b.child(a, cc)
            for d, bb in kk:
                c.children_spawned += 1
                kch = k.child(d, bb)
                r2 = (pnl.child(cc, d) if live[0] else None,
                      pml.child(a, d) if live[1] else None,
                      pns.child(cc, bb) if live[2] else None,
                      pms.child(a, bb) if live[3] else None)
                if self.spawn is not None and depth == 0:
                    self.spawn.append((bch, kch, r2, tuple(live)))
                else:
                    self.visit(bch, kch, r2, tuple(live), depth + 1)

    def contract(self, b, k, refs, live):
        c = self.c
        A = leaf_cache(b, self.shells, canonical=True)
        B = leaf_cache(k, self.shells, canonical=True)
        ma, mb = A["pd"].n, B["pd"].n
        sq_a, sq_b = np.sqrt(A["q"]), np.sqrt(B["q"])
        fa, fk = (sq_a, sq_b) if self.mode == "schwarz" else (A["q"], B["q"])
        src = (("fj", "nj", "fi", "ni"), ("fi", "ni", "fi", "ni"),
               ("fj", "nj", "fj", "nj"), ("fi", "ni", "fj", "nj"))
        masks = [None] * 4
        union = None
        for g in range(4):
            if not live[g]:
                continue
            s = src[g]
            pg = _pmax_block(self.P, A[s[0]], A[s[1]], B[s[2]], B[s[3]])
            bound = (fa[:, None] * pg) * fk[None, :]
            keep = bound > self.tau
            masks[g] = keep
            union = keep.copy() if union is None else (union | keep)
            ncull = ma * mb - int(keep.sum())
            if ncull:
                c.quartets_culled_leaf += ncull
                sb = bound if self.mode == "schwarz" else (sq_a[:, None] * pg) * sq_b[None, :]
                c.culled_bound_ledger += 0.5 * float(sb[~keep].sum())
        nkeep = int(union.sum())
        c.eri_shell_quartets += nkeep
        if not self.evaluate or nkeep == 0:
            return
        ia, ib = np.nonzero(union)
        blocks = eri_blocks(self.shells, A["pd"], B["pd"], ia, ib)
        if self.qlog is not None:
            self.qlog.extend(zip(A["pd"].i[ia].tolist(), A["pd"].j[ia].tolist(),
                                 B["pd"].i[ib].tolist(), B["pd"].j[ib].tolist()))
        wa, wb = A["wd"][ia], B["wd"][ib]
        specs = (("jk", "il", None), ("ik", "jl", wa), ("jl", "ik", wb), ("il", "jk", wa * wb))
        for g in range(4):
            if not live[g]:
                continue
            m = masks[g][ia, ib].astype(float)
            srcs, dst, w = specs[g]
            w = m if w is None else m * w
            _accumulate(self.K, self.P, blocks, ia, ib, A, B, srcs, dst, w)


def symmetrize_final(K, tol=1e-10):
    K = np.asarray(K, dtype=float)
    asym = float(np.abs(K - K.T).max()) if K.size else 0.0
    if asym > tol:
        raise LogicError(f"asymmetry {asym:.3e} exceeds {tol:.1e}")
    return 0.5 * (K + K.T)


def exchange_symmetric(shells, pairs, Ptree, P, tau=0.0, mode="schwarz",
                       quartet_log=None, evaluate=True, threads=1):
    """exchange_symmetry.py:364-409 restated (function-level for p shells)."""
    if tau < 0.0:
        raise InvalidArgumentError("tau_2e must be non-negative")
    if mode not in ("schwarz", "literal"):
        raise InvalidArgumentError(f"unknown screening mode {mode!r}")
    n = pairs.row.fhi
    want = quartet_log is not None
    run = _Sym(shells, P, n, tau, mode, evaluate, want)
    refs = (Ptree,) * 4
    alive = (True,) * 4
    if threads > 1:
        run.spawn = []
        run.visit(pairs, pairs, refs, alive, depth=0)

        def work(args):
            sub = _Sym(shells, P, n, tau, mode, evaluate, want)
            sub.visit(*args)
            return sub

        with ThreadPoolExecutor(max_workers=threads) as pool:
            subs = list(pool.map(work, run.spawn))
        for sub in subs:
            run.K += sub.K
            run.c.merge(sub.c)
            if want:
                run.qlog.extend(sub.qlog)
    else:
        run.visit(pairs, pairs, refs, alive)
    if want:
        quartet_log.extend(run.qlog)
    K = symmetrize_final(run.K) if evaluate else run.K
    return K, run.c


# --------------------------------------------------------------------------
# dense references (oracle.py:47-108)

def dense_exchange(shells, P):
    """Unscreened K over every shell quartet (oracle.py:47-66)."""
    n = sum(sh.nfn for sh in shells)
    ns = len(shells)
    K = np.zeros((n, n))
    plist = [(i, j) for i in range(ns) for j in range(ns)]
    pd = Pairs(shells, plist)
    fn = np.asarray([sh.fn for sh in shells])
    nf = np.asarray([sh.nfn for sh in shells])
    cache = {"fi": fn[pd.i], "fj": fn[pd.j], "ni": nf[pd.i], "nj": nf[pd.j]}
    allp = np.arange(pd.n)
    for a in range(pd.n):
        blocks = eri_blocks(shells, pd, pd, np.full(pd.n, a), allp)
        _accumulate(K, P, blocks, np.full(pd.n, a), allp, cache, cache, "jk", "il", None)
    return K


def screened_quartets(shells, P, tau, mode="schwarz"):
    """Direct-SCF keep set (oracle.py:69-99): bound = (f(Q_ij)|P_jk|)f(Q_kl) > tau."""
    ns = len(shells)
    plist = [(i, j) for i in range(ns) for j in range(ns)]
    canon = Pairs(shells, [(min(i, j), max(i, j)) for i, j in plist])
    q = diagonal_q(shells, canon).reshape(ns, ns)
    fq = np.sqrt(q) if mode == "schwarz" else q
    fn = np.asarray([sh.fn for sh in shells])
    nf = np.asarray([sh.nfn for sh in shells])
    pm = _pmax_block(P, fn, nf, fn, nf)
    bound = (fq[:, :, None, None] * pm[None, :, :, None]) * fq[None, None, :, :]
    keep = bound > tau
    return keep, bound


def dense_exchange_screened(shells, P, tau, mode="schwarz", quartet_log=None):
    ns = len(shells)
    keep, bound = screened_quartets(shells, P, tau, mode)
    skipped = 0.5 * float(bound[~keep].sum())
    idx = np.argwhere(keep)
    n = sum(sh.nfn for sh in shells)
    K = np.zeros((n, n))
    plist = [(i, j) for i in range(ns) for j in range(ns)]
    pd = Pairs(shells, plist)
    fn = np.asarray([sh.fn for sh in shells])
    nf = np.asarray([sh.nfn for sh in shells])
    cache = {"fi": fn[pd.i], "fj": fn[pd.j], "ni": nf[pd.i], "nj": nf[pd.j]}
    for lo in range(0, len(idx), 100000):
        part = idx[lo:lo + 100000]
        i, j, k, l = part.T
        ia, ib = i * ns + j, k * ns + l
        blocks = eri_blocks(shells, pd, pd, ia, ib)
        _accumulate(K, P, blocks, ia, ib, cache, cache, "jk", "il", None)
    if quartet_log is not None:
        quartet_log.extend(map(tuple, idx.tolist()))
    return K, skipped


# --------------------------------------------------------------------------
# one-call convenience used by tests / bench

class Setup:
    """Everything the drivers consume, built by the oracle from a system."""

    def __init__(self, system, P, tau_ovlp=0.0, leaf_size=10, zero_drop=0.0):
        self.shells = as_oracle_shells(system)
        self.P = np.asarray(P, dtype=float)
        self.root = build_partition([sh.nfn for sh in self.shells], leaf_size)
        self.s_abs = np.abs(overlap_matrix(self.shells))
        self.pairs = build_pair_tree(self.shells, self.root, tau_ovlp, self.s_abs)
        self.Ptree = build_matrix_tree(self.P, self.root, zero_drop)

    def naive(self, tau, **kw):
        return exchange_naive(self.shells, self.pairs, self.pairs, self.Ptree, self.P, tau, **kw)

    def symmetric(self, tau, **kw):
        return exchange_symmetric(self.shells, self.pairs, self.Ptree, self.P, tau, **kw)


def span_levels(root):
    """Span lists per level; ragged leaves repeat (quadtree.py:59-70)."""
    out = []
    fr = [root]
    while True:
        out.append(fr)
        if all(s.is_leaf for s in fr):
            return out
        fr = [c for s in fr for c in s.kids()]
