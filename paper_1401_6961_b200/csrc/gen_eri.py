"""Generate eri_classes.cuh: straight-line Obara-Saika / HGP code per class.

For each angular class (la, lb, lc, ld) in {0,1}^4 this emits

    struct Eri<la,lb,lc,ld> {
        static constexpr int NI, NJ, NK, NL, L;
        __device__ static void eval(bra, nb, ket, nk, A, B, C, D, tab, out);
    };

where bra[0:nb] / ket[0:nk] are the primitive pairs of the bra / ket shell
pair (PrimPair tables of hxf_internal.cuh) and tab the Boys table of order L.
Per primitive quartet: Boys F_0..F_L, vertical recursion (electron 1 on P,
electron 2 on Q, as in the CPU oracle's ``eri_general``) onto [e0|f0];
contraction in registers; then the horizontal transfer
(a,b+1_i| = (a+1_i,b| + AB_i (a,b| on the contracted values.
Output layout out[((i*NJ + j)*NK + k)*NL + l], p components ordered x,y,z.

Far-field quartets (every primitive quartet's Boys argument T above the
table range, decided per quartet in leaf.cu) run core<NKC, true>: the
asymptotic F_m only (boys_far, the same values the branch-free evaluation
selects there), and for (ss|ss) the closed form c'_b c'_k sqrt(pi)/2 / |P-Q|
with c' = c / sqrt(p) stored per primitive pair (PrimPair.cs).

Light classes (L <= 1) get a compile-time ket primitive count: eval()
dispatches on nk (warp-uniform, survivors are sorted by primitive counts) to
core<NKC>, which caches the ket primitives in registers and fully unrolls the
ket loop without branches, so the independent primitive-quartet chains can
be interleaved (instruction-level parallelism).

Run:  python gen_eri.py > eri_classes.cuh      (python gen_eri.py --flops: flop table)
"""

import itertools
import sys

UNIT = ((1, 0, 0), (0, 1, 0), (0, 0, 1))
ZERO = (0, 0, 0)
AX = "xyz"
MAXK = 9


def carts(l):
    return [ZERO] if l == 0 else list(UNIT)


def carts_upto(lo, hi):
    out = []
    for L in range(lo, hi + 1):
        for x in range(L, -1, -1):
            for y in range(L - x, -1, -1):
                out.append((x, y, L - x - y))
    return out


def sub(v, i):
    return v[:i] + (v[i] - 1,) + v[i + 1:]


def add(v, i):
    return v[:i] + (v[i] + 1,) + v[i + 1:]


def name(v):
    return "".join(str(c) for c in v)


class Gen:
    def __init__(self):
        self.lines = []
        self.memo = {}
        self.n = 0

    def tmp(self, expr, prefix="t"):
        v = f"{prefix}{self.n}"
        self.n += 1
        self.lines.append(f"const double {v} = {expr};")
        return v

    def vrr(self, e, f, m):
        key = (e, f, m)
        if key in self.memo:
            return self.memo[key]
        if e == ZERO and f == ZERO:
            v = f"bm{m}"
        elif e != ZERO:
            i = next(t for t in range(3) if e[t] > 0)
            e1 = sub(e, i)
            a = self.vrr(e1, f, m)
            b = self.vrr(e1, f, m + 1)
            expr = f"PA{AX[i]} * {a} + WP{AX[i]} * {b}"
            if e1[i] > 0:
                e2 = sub(e1, i)
                c = self.vrr(e2, f, m)
                d = self.vrr(e2, f, m + 1)
                expr += f" + {float(e1[i])} * o2p * ({c} - rp * {d})"
            if f[i] > 0:
                g = self.vrr(e1, sub(f, i), m + 1)
                expr += f" + {float(f[i])} * o2pq * {g}"
            v = self.tmp(expr)
        else:
            i = next(t for t in range(3) if f[t] > 0)
            f1 = sub(f, i)
            a = self.vrr(e, f1, m)
            b = self.vrr(e, f1, m + 1)
            expr = f"QC{AX[i]} * {a} + WQ{AX[i]} * {b}"
            if f1[i] > 0:
                f2 = sub(f1, i)
                c = self.vrr(e, f2, m)
                d = self.vrr(e, f2, m + 1)
                expr += f" + {float(f1[i])} * o2q * ({c} - rq * {d})"
            v = self.tmp(expr)
        self.memo[key] = v
        return v


def prim_body(w, la, lb, lc, ld, accs, ind, fold=False):
    """Statements for one primitive quartet (bp, kp in scope).  FAR (a template
    parameter of core) selects the asymptotic Boys branch only (boys_far)."""
    L = la + lb + lc + ld
    p = " " * ind
    if L == 0 and fold:  # (ss|ss) far: c'_b c'_k sqrt(pi)/2 / |P - Q| (c' = c / sqrt(p), PrimPair.cs)
        w(p + "if constexpr (FAR) {")
        w(p + "  const double PQx = bp.x - kp.x, PQy = bp.y - kp.y, PQz = bp.z - kp.z;")
        w(p + "  const double R2 = PQx * PQx + PQy * PQy + PQz * PQz;")
        w(p + "  accb = fma(kp.cs, rsqrt_pos(R2), accb);")
        w(p + "} else {")
        prim_body_ss(w, p + "  ")
        w(p + "}")
        return
    w(p + "const double ps = bp.p + kp.p;")
    w(p + "const double r = rsqrt_pos(ps);")
    w(p + "const double r2 = r * r;")
    w(p + "const double PQx = bp.x - kp.x, PQy = bp.y - kp.y, PQz = bp.z - kp.z;")
    w(p + "const double R2 = PQx * PQx + PQy * PQy + PQz * PQz;")
    w(p + "const double T = bp.p * kp.p * r2 * R2;")
    w(p + "const double pref = bp.c * kp.c * r;")
    w(p + f"double F[{L + 1}];")
    w(p + "if constexpr (FAR) {")
    w(p + f"  boys_far<{L}>(T, F);")
    w(p + "} else {")
    w(p + f"  boys_eval<{L}>(T, F, tab);")
    w(p + "}")
    prim_rest(w, la, lb, lc, ld, accs, p)


def prim_body_ss(w, p):
    if True:  # (ss|ss): bra coefficient applied once per bra primitive (accb)
        w(p + "const double ps = bp.p + kp.p;")
        w(p + "const double r = rsqrt_pos(ps);")
        w(p + "const double PQx = bp.x - kp.x, PQy = bp.y - kp.y, PQz = bp.z - kp.z;")
        w(p + "const double R2 = PQx * PQx + PQy * PQy + PQz * PQz;")
        w(p + "const double T = bp.p * kp.p * (r * r) * R2;")
        w(p + "double F[1];")
        w(p + "boys_eval<0>(T, F, tab);")
        w(p + "accb = fma(kp.c * r, F[0], accb);")


def prim_rest(w, la, lb, lc, ld, accs, p):
    L = la + lb + lc + ld
    for m in range(L + 1):
        w(p + f"const double bm{m} = pref * F[{m}];")
    if L > 0:
        if la + lb > 0:
            w(p + "const double rp = kp.p * r2;")
            w(p + "const double WPx = -rp * PQx, WPy = -rp * PQy, WPz = -rp * PQz;")
        if lc + ld > 0:
            w(p + "const double rq = bp.p * r2;")
            w(p + "const double WQx = rq * PQx, WQy = rq * PQy, WQz = rq * PQz;")
            w(p + "const double QCx = kp.x - C.x, QCy = kp.y - C.y, QCz = kp.z - C.z;")
            w(p + "const double o2q = 0.5 * kp.ip;")
        if la + lb > 0 and lc + ld > 0:
            w(p + "const double o2pq = 0.5 * r2;")
    g = Gen()
    res = {}
    for e, f in accs:
        res[(e, f)] = g.vrr(e, f, 0)
    for line in g.lines:
        w(p + line)
    for e, f in accs:
        w(p + f"acc_{name(e)}_{name(f)} += {res[(e, f)]};")


def gen_class(la, lb, lc, ld):
    L = la + lb + lc + ld
    es = carts_upto(la, la + lb)
    fs = carts_upto(lc, lc + ld)
    ni, nj, nk, nl = (len(carts(x)) for x in (la, lb, lc, ld))
    accs = [(e, f) for e in es for f in fs]
    cached = L <= 1
    need_ip = lc + ld > 0
    # (ss|ss) far path reads only {cs, x, y, z}
    load = "(FAR ? load_pp_far : load_pp)" if L == 0 else "load_pp"
    out = []
    w = out.append
    w(f"template <> struct Eri<{la},{lb},{lc},{ld}> {{")
    w(f"  static constexpr int NI = {ni}, NJ = {nj}, NK = {nk}, NL = {nl}, L = {L};")
    # ---- core<NKC>: NKC > 0 compile-time ket primitive count (register cache)
    w("  template <int NKC, bool FAR>")
    w("  __device__ __forceinline__ static void core(const PrimPair* __restrict__ bra, int nb,")
    w("      const PrimPair* __restrict__ ket, int nk, const double3 A, const double3 B,")
    w("      const double3 C, const double3 D, const double* __restrict__ tab,")
    w("      double* __restrict__ out) {")
    for e, f in accs:
        w(f"    double acc_{name(e)}_{name(f)} = 0.0;")
    if cached:
        w("    if constexpr (NKC > 0) {")
        w("      PrimPair kq[NKC > 0 ? NKC : 1];")
        w("#pragma unroll")
        w(f"      for (int t = 0; t < NKC; ++t) kq[t] = {load}(ket + t);")
        w(f"      PrimPair bn = {load}(bra);")
        w("      for (int ib = 0; ib < nb; ++ib) {")
        w("        const PrimPair bp = bn;")
        w(f"        if (ib + 1 < nb) bn = {load}(bra + ib + 1);  // prefetch the next bra primitive")
        if la + lb > 0:
            w("        const double PAx = bp.x - A.x, PAy = bp.y - A.y, PAz = bp.z - A.z;")
            w("        const double o2p = 0.5 * bp.ip;")
        if L == 0:
            w("        double accb = 0.0;")
        w("#pragma unroll")
        w("        for (int ik = 0; ik < NKC; ++ik) {")
        w("          const PrimPair& kp = kq[ik];")
        prim_body(w, la, lb, lc, ld, accs, 10, fold=True)
        w("        }")
        if L == 0:
            w("        acc_000_000 = fma(FAR ? bp.cs : bp.c, accb, acc_000_000);")
        w("      }")
        w("    } else {")
    w("      for (int ib = 0; ib < nb; ++ib) {")
    w(f"        const PrimPair bp = {load}(bra + ib);")
    if la + lb > 0:
        w("        const double PAx = bp.x - A.x, PAy = bp.y - A.y, PAz = bp.z - A.z;")
        w("        const double o2p = 0.5 * bp.ip;")
    w(f"        PrimPair kn = {load}(ket);")
    if L == 0:
        w("        double accb = 0.0;")
    w("        for (int ik = 0; ik < nk; ++ik) {")
    w("          const PrimPair kp = kn;")
    w(f"          if (ik + 1 < nk) kn = {load}(ket + ik + 1);  // prefetch: hide the L1/L2 latency")
    prim_body(w, la, lb, lc, ld, accs, 10, fold=True)
    w("        }")
    if L == 0:
        w("        acc_000_000 = fma(FAR ? bp.cs : bp.c, accb, acc_000_000);")
    w("      }")
    if cached:
        w("    }")
    if L == 0:
        w("    if constexpr (FAR) acc_000_000 *= HALF_SQRT_PI;")
    # horizontal recursion on contracted values
    memo = {}
    hl = []
    cnt = [0]

    def hrr(a, b, c, d):
        key = (a, b, c, d)
        if key in memo:
            return memo[key]
        if b != ZERO:
            i = next(t for t in range(3) if b[t] > 0)
            b1 = sub(b, i)
            x = hrr(add(a, i), b1, c, d)
            y = hrr(a, b1, c, d)
            v = f"h{cnt[0]}"
            cnt[0] += 1
            hl.append(f"const double {v} = {x} + AB{AX[i]} * {y};")
        elif d != ZERO:
            i = next(t for t in range(3) if d[t] > 0)
            d1 = sub(d, i)
            x = hrr(a, b, add(c, i), d1)
            y = hrr(a, b, c, d1)
            v = f"h{cnt[0]}"
            cnt[0] += 1
            hl.append(f"const double {v} = {x} + CD{AX[i]} * {y};")
        else:
            v = f"acc_{name(a)}_{name(c)}"
        memo[key] = v
        return v

    outs = []
    for (x, a), (y, b), (z, c), (t, d) in itertools.product(
            enumerate(carts(la)), enumerate(carts(lb)), enumerate(carts(lc)), enumerate(carts(ld))):
        outs.append((((x * nj + y) * nk + z) * nl + t, hrr(a, b, c, d)))
    if lb:
        w("    const double ABx = A.x - B.x, ABy = A.y - B.y, ABz = A.z - B.z;")
    if ld:
        w("    const double CDx = C.x - D.x, CDy = C.y - D.y, CDz = C.z - D.z;")
    for line in hl:
        w("    " + line)
    for idx, v in outs:
        w(f"    out[{idx}] = {v};")
    w("  }")
    # ---- eval: dispatch on the (warp-uniform) ket primitive count
    w("  template <bool FAR>")
    w("  __device__ __forceinline__ static void eval(const PrimPair* __restrict__ bra, int nb,")
    w("      const PrimPair* __restrict__ ket, int nk, const double3 A, const double3 B,")
    w("      const double3 C, const double3 D, const double* __restrict__ tab,")
    w("      double* __restrict__ out) {")
    if cached:
        w("    switch (nk) {")
        for k in range(1, MAXK + 1):
            w(f"      case {k}: core<{k}, FAR>(bra, nb, ket, nk, A, B, C, D, tab, out); return;")
        w("      default: core<0, FAR>(bra, nb, ket, nk, A, B, C, D, tab, out); return;")
        w("    }")
    else:
        w("    core<0, FAR>(bra, nb, ket, nk, A, B, C, D, tab, out);")
    w("  }")
    w("};")
    del need_ip
    return "\n".join(out)


def _ops(expr):
    return expr.count("*") + expr.count("+") + expr.count(" - ")


def flop_counts(la, lb, lc, ld):
    """Algorithmic FP64 flops of the scheme: (per primitive quartet, per shell quartet).

    The all-s class uses the SURVEY.md 8(d) contract of 30 flops per primitive
    quartet (integrals.py:157-165 with precomputed pair tables, F0 at a fixed
    11).  Other classes add, per primitive quartet, the vertical-recursion
    operations as generated plus 3 per extra F_m (downward recursion), the
    W/Q-centre set-up (WP, WQ, QC: 3-6 each, 1/2p-type factors: 1 each);
    per shell quartet the horizontal transfer.
    """
    L = la + lb + lc + ld
    g = Gen()
    es = carts_upto(la, la + lb)
    fs = carts_upto(lc, lc + ld)
    for e in es:
        for f in fs:
            g.vrr(e, f, 0)
    per_prim = 30 + len(es) * len(fs) - 1
    if L:
        per_prim += 3 * L + L  # F_m recursion + bm scaling
        per_prim += sum(_ops(line.split("=", 1)[1]) for line in g.lines)
        if la + lb:
            per_prim += 3 + 1 + 1 + 1    # PA (per bra prim, amortised as 1/kb), WP, o2p, rp
        if lc + ld:
            per_prim += 3 + 3 + 1 + 1    # WQ, QC, o2q, rq
        if la + lb and lc + ld:
            per_prim += 1
    n_out = len(carts(la)) * len(carts(lb)) * len(carts(lc)) * len(carts(ld))
    per_quartet = 2 * 3 * (lb + ld) + 2 * max(0, n_out - 1) * (1 if (lb or ld) else 0)
    return per_prim, per_quartet


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--flops":
        import json
        tab = {}
        for cls in itertools.product((0, 1), repeat=4):
            idx = (cls[0] << 3) | (cls[1] << 2) | (cls[2] << 1) | cls[3]
            tab[idx] = flop_counts(*cls)
        print(json.dumps({"per_prim": [tab[k][0] for k in range(16)],
                          "per_quartet": [tab[k][1] for k in range(16)]}))
        return
    print("// generated by gen_eri.py -- do not edit")
    print("#pragma once")
    print("// boys_eval: boys_bf (Schwarz factors, trees.cu) or boys_bf_scaled (ERI kernels, leaf.cu),")
    print("// chosen by the including translation unit")
    print("template <int LA, int LB, int LC, int LD> struct Eri;")
    for cls in itertools.product((0, 1), repeat=4):
        print(gen_class(*cls))
        print()


if __name__ == "__main__":
    main()
