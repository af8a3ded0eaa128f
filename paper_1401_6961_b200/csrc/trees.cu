// Device construction of the shell-pair and density quadtrees (SURVEY.md
// kernels K1-K3).  Restates quadtree.py:198-337 of the reference:
//   - s-proxy contracted overlap, block max |S| per leaf pair node, pruning
//     pruned <=> block max |S| < tau_ovlp (quadtree.py:298-301, 323-327);
//   - primitive pair tables per ordered shell pair of live leaf nodes
//     (integrals.py:115-154);
//   - Q_ij = (ij|ij) in canonical (min,max) orientation (quadtree.py:307-313),
//     max over function pairs for p shells;
//   - node norms with correctly rounded fsum (quadtree.py:20-25), row/column
//     sum maxima (quadtree.py:314-316, 328-334);
//   - density norms / absent flags (quadtree.py:210-235).
// Node arrays are dense per level: node (r, c) of level L lives at
// node_off[L] + r * n_L + c; a partition leaf repeats at deeper levels.

#include <cub/cub.cuh>

#include "boys.cuh"
#include "hxf_internal.cuh"
#define boys_eval boys_bf  // Schwarz factors: the reference Boys evaluation
#include "eri_classes.cuh"

#define SQRT_TWO_PI_POW_2_5 5.914967172795613 /* sqrt(2 pi^{5/2}) */

namespace {

// numpy pairwise summation order for short contiguous vectors
// (pairwise_sum: < 8 sequential, else 8 accumulators then the remainder).
__device__ double np_sum(const double* v, int n, int stride) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r = __dadd_rn(r, v[i * stride]);
        return r;
    }
    double a[8];
    for (int j = 0; j < 8; ++j) a[j] = v[j * stride];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) a[j] = __dadd_rn(a[j], v[(i + j) * stride]);
    double r = __dadd_rn(__dadd_rn(__dadd_rn(a[0], a[1]), __dadd_rn(a[2], a[3])),
                         __dadd_rn(__dadd_rn(a[4], a[5]), __dadd_rn(a[6], a[7])));
    for (; i < n; ++i) r = __dadd_rn(r, v[i * stride]);
    return r;
}

// contracted s(-proxy) overlap of shells a <= b (integrals.py:58-64)
__device__ double overlap_s(const DevBasis& B, int a, int b) {
    const double3 A = B.ctr[a], C = B.ctr[b];
    const double dx = A.x - C.x, dy = A.y - C.y, dz = A.z - C.z;
    const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const int a0 = B.poff[a], a1 = B.poff[a + 1], b0 = B.poff[b], b1 = B.poff[b + 1];
    double terms[9];
    int n = 0;
    for (int i = a0; i < a1; ++i)
        for (int j = b0; j < b1; ++j) {
            const double ea = B.exps[i], eb = B.exps[j];
            const double p = __dadd_rn(ea, eb);
            const double s = __dmul_rn(pow(__ddiv_rn(M_PI, p), 1.5),
                                       exp(__dmul_rn(__ddiv_rn(-__dmul_rn(ea, eb), p), r2)));
            terms[n++] = __dmul_rn(__dmul_rn(B.sw[i], B.sw[j]), s);
        }
    return np_sum(terms, n, 1);
}

__global__ void k_leaf_smax(DevBasis B, DevLevels lv, const int* lslo, const int* lshi, int nleaf,
                            double* smax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    if (r > c) return;
    double m = 0.0;
    for (int i = lslo[r]; i < lshi[r]; ++i)
        for (int j = lslo[c]; j < lshi[c]; ++j) {
            const double s = fabs(i <= j ? overlap_s(B, i, j) : overlap_s(B, j, i));
            m = fmax(m, s);
        }
    smax[(int64_t)r * nleaf + c] = m;
    smax[(int64_t)c * nleaf + r] = m;
}

// overlap_matrix override (quadtree.py:284-293): block max of the caller's |S|
// over the leaf spans (r, c), both orientations (not assumed symmetric)
__global__ void k_leaf_smax_user(const double* __restrict__ S, int ns, const int* lslo, const int* lshi, int nleaf,
                                 double* smax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    double m = 0.0;
    for (int i = lslo[r]; i < lshi[r]; ++i)
        for (int j = lslo[c]; j < lshi[c]; ++j) m = fmax(m, fabs(S[(int64_t)i * ns + j]));
    smax[t] = m;
}

__global__ void k_leaf_pair_counts(const double* smax, double tau, const int* lslo,
                                   const int* lshi, const int* lplo, const int* lphi, int nleaf,
                                   int64_t* npairs, int64_t* nprims) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    const bool live = !(smax[t] < tau);
    npairs[t] = live ? (int64_t)(lshi[r] - lslo[r]) * (lshi[c] - lslo[c]) : 0;
    nprims[t] = live ? (int64_t)(lphi[r] - lplo[r]) * (lphi[c] - lplo[c]) : 0;
}

// one thread per live leaf pair node: fill pair ids, prim pair tables
__global__ void k_fill_pairs(DevBasis B, const double* smax, double tau, const int* lslo,
                             const int* lshi, int nleaf, const int64_t* pbase,
                             const int64_t* ppbase, int64_t* leaf_base, int* pi, int* pj,
                             int64_t* ppoff, PrimPair* pp, int4* info) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    if (smax[t] < tau) {
        leaf_base[t] = -1;
        return;
    }
    int64_t pid = pbase[t];
    int64_t po = ppbase[t];
    leaf_base[t] = pid;
    for (int i = lslo[r]; i < lshi[r]; ++i)
        for (int j = lslo[c]; j < lshi[c]; ++j, ++pid) {
            pi[pid] = i;
            pj[pid] = j;
            ppoff[pid] = po;
            info[pid] = make_int4(B.fn[i], B.fn[j], (int)po,
                                  (B.poff[i + 1] - B.poff[i]) * (B.poff[j + 1] - B.poff[j]));
            const double3 A = B.ctr[i], C = B.ctr[j];
            const double dx = A.x - C.x, dy = A.y - C.y, dz = A.z - C.z;
            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            for (int a = B.poff[i]; a < B.poff[i + 1]; ++a)
                for (int b = B.poff[j]; b < B.poff[j + 1]; ++b, ++po) {
                    const double ea = B.exps[a], eb = B.exps[b];
                    const double p = __dadd_rn(ea, eb);
                    const double w = __dmul_rn(__dmul_rn(B.w[a], B.w[b]),
                                               exp(__dmul_rn(__ddiv_rn(-__dmul_rn(ea, eb), p), r2)));
                    PrimPair q;
                    q.p = p;
                    q.ip = 1.0 / p;
                    q.c = w * q.ip * SQRT_TWO_PI_POW_2_5;
                    q.x = __ddiv_rn(__dadd_rn(__dmul_rn(ea, A.x), __dmul_rn(eb, C.x)), p);
                    q.y = __ddiv_rn(__dadd_rn(__dmul_rn(ea, A.y), __dmul_rn(eb, C.y)), p);
                    q.z = __ddiv_rn(__dadd_rn(__dmul_rn(ea, A.z), __dmul_rn(eb, C.z)), p);
                    q.cs = q.c * sqrt(q.ip);
                    q.pad1 = 0.0;
                    pp[po] = q;
                }
        }
    if (r == nleaf - 1 && c == nleaf - 1) ppoff[pid] = po;
}

template <int LA, int LB>
__device__ double diag_q(const PrimPair* pp, int64_t b0, int64_t b1, double3 A, double3 Bc) {
    typedef Eri<LA, LB, LA, LB> E;
    double out[E::NI * E::NJ * E::NK * E::NL];
    E::template eval<false>(pp, (int)(b1 - b0), pp, (int)(b1 - b0), A, Bc, A, Bc, boys_table_global(E::L), out);
    double q = 0.0;
    for (int x = 0; x < E::NI; ++x)
        for (int y = 0; y < E::NJ; ++y) q = fmax(q, out[((x * E::NJ + y) * E::NK + x) * E::NL + y]);
    return q;
}

// Q for canonical pairs i <= j, mirrored to (j, i) (quadtree.py:307-313).  With a
// caller-supplied, non-symmetric |S| (the overlap_matrix override) a node can be
// live while its mirror is pruned: the mirror write is skipped when the (j, i)
// node is pruned, and a pair (i > j) whose canonical node is pruned evaluates
// its own Q from its primitive pairs transposed into the canonical (j, i) order,
// so the value is bitwise the one the canonical node would have cached.
__device__ double diag_q_any(int li, int lj, const PrimPair* pp, int n, double3 A, double3 C) {
    if (li == 0 && lj == 0) return diag_q<0, 0>(pp, 0, n, A, C);
    if (li == 0) return diag_q<0, 1>(pp, 0, n, A, C);
    if (lj == 0) return diag_q<1, 0>(pp, 0, n, A, C);
    return diag_q<1, 1>(pp, 0, n, A, C);
}

__global__ void k_diag_q(DevBasis B, int64_t n_pairs, const int* pi, const int* pj,
                         const int64_t* ppoff, const PrimPair* pp, const int* leaf_of_shell,
                         const int* lslo, const int* lshi, int nleaf, const int64_t* leaf_base,
                         double* q) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const int i = pi[t], j = pj[t];
    const int Li = leaf_of_shell[i], Lj = leaf_of_shell[j];
    const int64_t mb = i == j ? -1 : leaf_base[(int64_t)Lj * nleaf + Li];   // the mirror pair's node
    const int64_t b0 = ppoff[t], b1 = ppoff[t + 1];
    const int n = (int)(b1 - b0);
    if (i > j) {
        if (mb >= 0) return;   // the canonical pair (j, i) exists and writes both
        const int ni = B.poff[i + 1] - B.poff[i], nj = B.poff[j + 1] - B.poff[j];
        // n <= 9: shells hold 1..3 primitives (hxf_system_create checks)
        PrimPair tr[16];       // (b over j outer, a over i inner): the (j, i) pair's order
        for (int a = 0; a < ni; ++a)
            for (int b = 0; b < nj; ++b) tr[b * ni + a] = pp[b0 + a * nj + b];
        q[t] = diag_q_any(B.l[j], B.l[i], tr, n, B.ctr[j], B.ctr[i]);
        return;
    }
    const double v = diag_q_any(B.l[i], B.l[j], pp + b0, n, B.ctr[i], B.ctr[j]);
    q[t] = v;
    // pair (j, i) lives in node (leaf(j), leaf(i)) at row j, column i
    if (mb >= 0) q[mb + (int64_t)(j - lslo[Lj]) * (lshi[Li] - lslo[Li]) + (i - lslo[Li])] = v;
}

// primitive Schwarz factors S = sqrt(max_comp (ab|ab)) of every primitive pair,
// and the ERI copy of each pair's primitives sorted by S, descending (ties by
// index), so a build can drop a negligible tail by shortening the count
//
// Far-field collapse: a pair of two s shells on one centre is a sum of concentric
// spherical Gaussian charges; outside their extent (where every Boys argument is past
// the table range, i.e. exactly the quartets the far-field kernels take) its potential
// is that of one point charge sum_u c_u / sqrt(p_u) at the centre, independent of the
// exponents.  Such a pair gets one extra primitive at epp[n_prim + pair id] {centre,
// p = min_u p_u (keeps T above the far-field bound the classification proved), cs = the
// summed charge, c = cs sqrt(p)}: the far-field kernels read it instead of the list
// (the asymptotic recurrences cancel p term by term, so any p gives the same value to
// rounding).  Summed in epp order so mirrored pairs (i,j), (j,i) agree.
__global__ void k_prim_schwarz_sort(DevBasis B, int64_t n_pairs, const int* pi, const int* pj,
                                    const int64_t* ppoff, const PrimPair* pp, PrimPair* epp, double* eS,
                                    int64_t n_prim, int collapse, uint8_t* fcol) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const int i = pi[t], j = pj[t];
    const int64_t b0 = ppoff[t], b1 = ppoff[t + 1];
    const double3 A = B.ctr[i], C = B.ctr[j];
    const int li = B.l[i], lj = B.l[j];
    double sv[16];
    int idx[16];
    const int n = (int)(b1 - b0);
    for (int u = 0; u < n; ++u) {
        const PrimPair* q = pp + b0 + u;
        double v;
        if (li == 0 && lj == 0) v = diag_q<0, 0>(q, 0, 1, A, C);
        else if (li == 0) v = diag_q<0, 1>(q, 0, 1, A, C);
        else if (lj == 0) v = diag_q<1, 0>(q, 0, 1, A, C);
        else v = diag_q<1, 1>(q, 0, 1, A, C);
        const double sval = sqrt(v);
        int k = u;  // insertion sort, descending, stable
        while (k > 0 && sv[k - 1] < sval) {
            sv[k] = sv[k - 1];
            idx[k] = idx[k - 1];
            --k;
        }
        sv[k] = sval;
        idx[k] = u;
    }
    for (int u = 0; u < n; ++u) {
        epp[b0 + u] = pp[b0 + idx[u]];
        eS[b0 + u] = sv[u];
    }
    const bool same = A.x == C.x && A.y == C.y && A.z == C.z;
    const bool col = collapse && li == 0 && lj == 0 && same && n > 1;
    fcol[t] = col ? 1 : 0;
    PrimPair f = pp[b0 + idx[0]];
    if (col) {
        double cs = 0.0, pmin = f.p;
        for (int u = 0; u < n; ++u) {
            const PrimPair& q = pp[b0 + idx[u]];
            cs += q.cs;
            pmin = fmin(pmin, q.p);
        }
        f.x = A.x; f.y = A.y; f.z = A.z;
        f.p = pmin;
        f.ip = 1.0 / pmin;
        f.cs = cs;
        f.c = cs * sqrt(pmin);
    }
    epp[n_prim + t] = f;
}

// Far-field geometry per pair (the ERI stage's per-quartet asymptotic test,
// leaf.cu): centroid c of the primitive centres, radius r with every centre
// within r of c, and ip = max 1/p, all as floats rounded outward (r and ip up,
// r also absorbs the centroid's float rounding), so that for any primitive
// pair b of a bra pair and k of a ket pair |P_b - Q_k| >= |c_B - c_K| - r_B - r_K
// and 1/p_b + 1/q_k <= ip_B + ip_K.
__global__ void k_pair_geo(int64_t n_pairs, const int64_t* ppoff, const PrimPair* pp, float4* geo, float* gip) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const int64_t b0 = ppoff[t], b1 = ppoff[t + 1];
    double cx = 0.0, cy = 0.0, cz = 0.0, ip = 0.0;
    for (int64_t u = b0; u < b1; ++u) {
        cx += pp[u].x;
        cy += pp[u].y;
        cz += pp[u].z;
        ip = fmax(ip, pp[u].ip);
    }
    const double inv = 1.0 / (double)(b1 - b0);
    const float fx = (float)(cx * inv), fy = (float)(cy * inv), fz = (float)(cz * inv);
    double r = 0.0;
    for (int64_t u = b0; u < b1; ++u) {
        const double dx = pp[u].x - fx, dy = pp[u].y - fy, dz = pp[u].z - fz;
        r = fmax(r, sqrt(dx * dx + dy * dy + dz * dz));
    }
    geo[t] = make_float4(fx, fy, fz, __double2float_ru(r * (1.0 + 1e-6) + 1e-4));
    gip[t] = __double2float_ru(ip * (1.0 + 1e-6));
}

// per pair: sqrt(Q) once (screening uses it for every quartet) and the class /
// primitive-count byte of the survivor sort key
__global__ void k_pair_meta(DevBasis B, int64_t n_pairs, const int* pi, const int* pj,
                            const double* q, double* sq, uint8_t* meta) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const int i = pi[t], j = pj[t];
    sq[t] = sqrt(q[t]);
    const int np = (B.poff[i + 1] - B.poff[i]) * (B.poff[j + 1] - B.poff[j]);
    meta[t] = (uint8_t)((B.l[i] << 1) | B.l[j] | ((np - 1) << 2));
}

// shell-level max |P| over each function block (|P_jk| for s shells): the
// per-quartet density factor of the leaf test
__global__ void k_shell_pmax(DevBasis B, const double* P, double* pmax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)B.ns * B.ns) return;
    const int s = (int)(t / B.ns), u = (int)(t % B.ns);
    const int f0 = B.fn[s], g0 = B.fn[u];
    double m = 0.0;
    for (int x = 0; x < B.nf[s]; ++x)
        for (int y = 0; y < B.nf[u]; ++y) m = fmax(m, fabs(P[(int64_t)(f0 + x) * B.nfn + g0 + y]));
    pmax[t] = m;
}

// leaf pair node norms: diag_norm = sqrt(fsum(Q^2)), row/col sum maxima
__global__ void k_leaf_norms(const int* lslo, const int* lshi, int nleaf, const int64_t* leaf_base,
                             const double* q, double* lnorm, double* lrow, double* lcol) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    const int64_t b = leaf_base[t];
    if (b < 0) {
        lnorm[t] = -1.0;
        lrow[t] = 0.0;
        lcol[t] = 0.0;
        return;
    }
    const int nr = lshi[r] - lslo[r], nc = lshi[c] - lslo[c];
    const double* Q = q + b;
    FSum fs;
    for (int k = 0; k < nr * nc; ++k) fs.add(__dmul_rn(Q[k], Q[k]));
    lnorm[t] = sqrt(fs.result());
    double rm = -INFINITY, cm = -INFINITY;
    for (int x = 0; x < nr; ++x) rm = fmax(rm, np_sum(Q + x * nc, nc, 1));
    for (int y = 0; y < nc; ++y) {
        double s = 0.0;
        for (int x = 0; x < nr; ++x) s = __dadd_rn(s, Q[x * nc + y]);
        cm = fmax(cm, s);
    }
    lrow[t] = rm;
    lcol[t] = cm;
}

// overlap-pruning comparisons (block max |S| < tau_ovlp) within 1e-12 relative of tau_ovlp
__global__ void k_overlap_ties(const double* smax, int n, int level, double tau, TieLog tl) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * n) return;
    const double m = smax[t];
    if (fabs(m - tau) <= 1e-12 * tau) {
        tie_emit(tl, HXF_TIE_OVERLAP, level, 0, !(m < tau), (int)(t / n), (int)(t % n), -1, -1, m, tau);
    }
}

// fill one level of the pair tree (bottom-up); leaves copy leaf-pair data
__global__ void k_pair_level(int level, int n, int nnext, const int* span_base_L,
                             const int* leaf_id, const int* kid0, const int* kid1, int nleaf,
                             const double* lnorm, const double* lrow, const double* lcol,
                             const double* lsmax, double tau, const int64_t* node_off,
                             double* norm, double* rowsum, double* colsum, double* smax) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * n) return;
    const int r = (int)(t / n), c = (int)(t % n);
    const int sr = span_base_L[0] + r, sc = span_base_L[0] + c;
    const int64_t me = node_off[level] + t;
    const int lr = leaf_id[sr], lc = leaf_id[sc];
    if (lr >= 0 && lc >= 0) {
        const int64_t k = (int64_t)lr * nleaf + lc;
        norm[me] = lnorm[k];
        rowsum[me] = lrow[k];
        colsum[me] = lcol[k];
        smax[me] = lsmax[k];
        return;
    }
    const int ra[2] = {kid0[sr], kid1[sr]}, ca[2] = {kid0[sc], kid1[sc]};
    const int na = ra[1] < 0 ? 1 : 2, nb = ca[1] < 0 ? 1 : 2;
    double m = 0.0;
    FSum fs;
    bool any_live = false;
    for (int a = 0; a < na; ++a)
        for (int b = 0; b < nb; ++b) {
            const int64_t ch = node_off[level + 1] + (int64_t)ra[a] * nnext + ca[b];
            m = fmax(m, smax[ch]);
            if (norm[ch] >= 0.0) {
                any_live = true;
                fs.add(__dmul_rn(norm[ch], norm[ch]));
            }
        }
    smax[me] = m;
    if (m < tau || !any_live) {
        norm[me] = -1.0;
        rowsum[me] = 0.0;
        colsum[me] = 0.0;
        return;
    }
    norm[me] = sqrt(fs.result());
    double rm = -INFINITY, cm = -INFINITY;
    for (int a = 0; a < na; ++a) {
        FSum s;
        for (int b = 0; b < nb; ++b) s.add(rowsum[node_off[level + 1] + (int64_t)ra[a] * nnext + ca[b]]);
        rm = fmax(rm, s.result());
    }
    for (int b = 0; b < nb; ++b) {
        FSum s;
        for (int a = 0; a < na; ++a) s.add(colsum[node_off[level + 1] + (int64_t)ra[a] * nnext + ca[b]]);
        cm = fmax(cm, s.result());
    }
    rowsum[me] = rm;
    colsum[me] = cm;
}

// density leaf blocks: present iff any nonzero and norm > zero_drop
__global__ void k_density_leaves(const double* P, int nfn, const int* lflo, const int* lfhi,
                                 int nleaf, double zero_drop, double* lnorm) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nleaf * nleaf) return;
    const int r = (int)(t / nleaf), c = (int)(t % nleaf);
    FSum fs;
    bool any = false;
    for (int x = lflo[r]; x < lfhi[r]; ++x)
        for (int y = lflo[c]; y < lfhi[c]; ++y) {
            const double v = P[(int64_t)x * nfn + y];
            any |= (v != 0.0);
            fs.add(__dmul_rn(v, v));
        }
    double nrm = sqrt(fs.result());
    lnorm[t] = (!any || nrm <= zero_drop) ? -1.0 : nrm;
}

__global__ void k_density_level(int level, int n, int nnext, const int* span_base_L,
                                const int* leaf_id, const int* kid0, const int* kid1, int nleaf,
                                const double* lnorm, const int64_t* node_off, double* norm) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)n * n) return;
    const int r = (int)(t / n), c = (int)(t % n);
    const int sr = span_base_L[0] + r, sc = span_base_L[0] + c;
    const int64_t me = node_off[level] + t;
    const int lr = leaf_id[sr], lc = leaf_id[sc];
    if (lr >= 0 && lc >= 0) {
        norm[me] = lnorm[(int64_t)lr * nleaf + lc];
    } else {
        const int ra[2] = {kid0[sr], kid1[sr]}, ca[2] = {kid0[sc], kid1[sc]};
        const int na = ra[1] < 0 ? 1 : 2, nb = ca[1] < 0 ? 1 : 2;
        FSum fs;
        bool any = false;
        for (int a = 0; a < na; ++a)
            for (int b = 0; b < nb; ++b) {
                const double v = norm[node_off[level + 1] + (int64_t)ra[a] * nnext + ca[b]];
                if (v >= 0.0) {
                    any = true;
                    fs.add(__dmul_rn(v, v));
                }
            }
        norm[me] = any ? sqrt(fs.result()) : -1.0;
    }
    // all-zero matrix: explicit root with norm 0 (quadtree.py:230-235)
    if (level == 0 && t == 0 && norm[me] < 0.0) norm[me] = 0.0;
}

// per live leaf pair node: row / column maxima of Q and row / column sums of
// sqrt(Q) over its shell pairs (the whole block), and for diagonal nodes also
// over the canonical triangle x <= y (the fourfold enumeration); fixed
// summation order (deterministic)
__global__ void k_node_vectors(const int* lslo, const int* lshi, int nl, const int64_t* leaf_base,
                               const int* ncid, const double* q, const double* sq, double* nvec,
                               double* nvec_tri) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= (int64_t)nl * nl) return;
    const int64_t bb = leaf_base[t];
    if (bb < 0) return;
    const int mu = (int)(t / nl), nu = (int)(t % nl);
    const int nmu = lshi[mu] - lslo[mu], nnu = lshi[nu] - lslo[nu];
    for (int tri = 0; tri < (mu == nu ? 2 : 1); ++tri) {
        double* v = tri ? nvec_tri + (int64_t)mu * NVEC : nvec + (int64_t)ncid[t] * NVEC;
        for (int k = 0; k < NVEC; ++k) v[k] = 0.0;
        for (int x = 0; x < nmu; ++x)
            for (int y = tri ? x : 0; y < nnu; ++y) {
                const int64_t pid = bb + x * nnu + y;
                const double qq = q[pid], s = sq[pid];
                v[NV_FR + x] = fmax(v[NV_FR + x], qq);
                v[NV_FC + y] = fmax(v[NV_FC + y], qq);
                v[NV_SR + x] += s;
                v[NV_SC + y] += s;
            }
        for (int k = 0; k < NV_MAXS; ++k) {
            v[NV_GR + k] = sqrt(v[NV_FR + k]);
            v[NV_GC + k] = sqrt(v[NV_FC + k]);
        }
    }
}

__global__ void k_live_flags(const int64_t* leaf_base, int64_t n, int* flag) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n) flag[t] = leaf_base[t] >= 0 ? 1 : 0;
}

__global__ void k_live_ids(const int64_t* leaf_base, int64_t n, int* ncid) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n && leaf_base[t] < 0) ncid[t] = -1;
}

__global__ void k_node_sqrts(int64_t n, const double* norm, const double* row, const double* col, double* snorm,
                             double* srow, double* scol) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const double v = norm[t];
    snorm[t] = v < 0.0 ? -1.0 : sqrt(v);
    srow[t] = sqrt(fmax(row[t], 0.0));
    scol[t] = sqrt(fmax(col[t], 0.0));
}

// per shell: sum of n_f(partner) sqrt(Q) over the pairs that contain it (K scale bound)
__global__ void k_pair_asum(DevBasis b, int64_t n, const int* pi, const int* pj, const double* sq, double* asum) {
    const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int i = pi[q], j = pj[q];
    const double v = sq[q];
    atomicAdd(asum + i, b.nf[j] * v);
    atomicAdd(asum + j, b.nf[i] * v);
}

__global__ void k_maxabs(const double* v, int64_t n, unsigned long long* out) {
    double m = 0.0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs(v[t]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

inline unsigned nblk(int64_t n, int b = 256) { return (unsigned)((n + b - 1) / b); }

template <typename T>
T* dalloc(size_t n, cudaStream_t st) {
    void* p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMallocAsync(&p, n * sizeof(T), st);
    if (e != cudaSuccess) throw HxfError{HXF_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e)};
    return (T*)p;
}

}  // namespace

// ---------------------------------------------------------------------------
// host orchestration

struct LeafTables {
    int* lslo;
    int* lshi;
    int* lplo;
    int* lphi;
    int* lflo;
    int* lfhi;
    int* leaf_of_shell;
};

static LeafTables make_leaf_tables(hxf_system* s, cudaStream_t st, std::vector<void*>& tmp) {
    const int nl = s->n_leaves;
    std::vector<int> slo(nl), shi(nl), plo(nl), phi(nl), flo(nl), fhi(nl), los(s->ns);
    const int D = s->n_levels - 1;
    for (int k = s->h_off[D]; k < s->h_off[D + 1]; ++k) {
        const int lid = s->h_leaf_id[k];
        slo[lid] = s->h_slo[k];
        shi[lid] = s->h_shi[k];
        flo[lid] = s->h_flo[k];
        fhi[lid] = s->h_fhi[k];
        plo[lid] = s->h_poff[slo[lid]];
        phi[lid] = s->h_poff[shi[lid]];
        for (int i = slo[lid]; i < shi[lid]; ++i) los[i] = lid;
    }
    LeafTables t;
    int** dst[] = {&t.lslo, &t.lshi, &t.lplo, &t.lphi, &t.lflo, &t.lfhi};
    std::vector<int>* src[] = {&slo, &shi, &plo, &phi, &flo, &fhi};
    for (int k = 0; k < 6; ++k) {
        *dst[k] = dalloc<int>(nl, st);
        tmp.push_back(*dst[k]);
        HXF_CUDA(cudaMemcpyAsync(*dst[k], src[k]->data(), nl * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    t.leaf_of_shell = dalloc<int>(s->ns, st);
    tmp.push_back(t.leaf_of_shell);
    HXF_CUDA(cudaMemcpyAsync(t.leaf_of_shell, los.data(), s->ns * sizeof(int), cudaMemcpyHostToDevice, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    return t;
}

void trees_build_pairs(hxf_pairs* pr, cudaStream_t st, const double* s_user) {
    NvtxRange nvtx_range("hxf: pair tree");
    hxf_system* s = pr->sys;
    std::vector<void*> tmp;
    const int nl = s->n_leaves;
    const int64_t nl2 = (int64_t)nl * nl;
    LeafTables lt = make_leaf_tables(s, st, tmp);
    double* lsmax = dalloc<double>(nl2, st);
    tmp.push_back(lsmax);
    if (s_user) { k_leaf_smax_user<<<nblk(nl2, 128), 128, 0, st>>>(s_user, s->ns, lt.lslo, lt.lshi, nl, lsmax); note_launch(); }
    else { k_leaf_smax<<<nblk(nl2, 128), 128, 0, st>>>(s->basis, s->lv, lt.lslo, lt.lshi, nl, lsmax); note_launch(); }
    int64_t* npairs = dalloc<int64_t>(nl2 + 1, st);
    int64_t* nprims = dalloc<int64_t>(nl2 + 1, st);
    int64_t* pbase = dalloc<int64_t>(nl2 + 1, st);
    int64_t* ppbase = dalloc<int64_t>(nl2 + 1, st);
    tmp.insert(tmp.end(), {npairs, nprims, pbase, ppbase});
    HXF_CUDA(cudaMemsetAsync(npairs + nl2, 0, sizeof(int64_t), st));
    HXF_CUDA(cudaMemsetAsync(nprims + nl2, 0, sizeof(int64_t), st));
    { k_leaf_pair_counts<<<nblk(nl2), 256, 0, st>>>(lsmax, pr->tau_ovlp, lt.lslo, lt.lshi, lt.lplo,
                                                  lt.lphi, nl, npairs, nprims); note_launch(); }
    size_t tb = 0;
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, npairs, pbase, nl2 + 1, st));
    void* tbuf = dalloc<char>(tb, st);
    tmp.push_back(tbuf);
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, npairs, pbase, nl2 + 1, st));
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, nprims, ppbase, nl2 + 1, st));
    int64_t tot[2];
    HXF_CUDA(cudaMemcpyAsync(&tot[0], pbase + nl2, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaMemcpyAsync(&tot[1], ppbase + nl2, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    pr->n_pairs = tot[0];
    pr->n_prim_pairs = tot[1];
    if (pr->n_pairs >= (1ll << 28))
        throw HxfError{HXF_EINVAL, "too many significant shell pairs for the 28-bit pair ids"};
    pr->leaf_base = dalloc<int64_t>(nl2, st);
    pr->pi = dalloc<int>(pr->n_pairs, st);
    pr->pj = dalloc<int>(pr->n_pairs, st);
    pr->ppoff = dalloc<int64_t>(pr->n_pairs + 1, st);
    pr->q = dalloc<double>(pr->n_pairs, st);
    pr->pp = dalloc<PrimPair>(pr->n_prim_pairs, st);
    pr->info = dalloc<int4>(pr->n_pairs, st);
    if (pr->n_prim_pairs >= (1ll << 31))
        throw HxfError{HXF_EINVAL, "too many primitive pairs for 32-bit offsets"};
    HXF_CUDA(cudaMemcpyAsync(pr->ppoff + pr->n_pairs, &tot[1], sizeof(int64_t), cudaMemcpyHostToDevice, st));
    { k_fill_pairs<<<nblk(nl2, 128), 128, 0, st>>>(s->basis, lsmax, pr->tau_ovlp, lt.lslo, lt.lshi, nl,
                                                 pbase, ppbase, pr->leaf_base, pr->pi, pr->pj,
                                                 pr->ppoff, pr->pp, pr->info); note_launch(); }
    HXF_CUDA(cudaMemcpyAsync(pr->ppoff + pr->n_pairs, &tot[1], sizeof(int64_t), cudaMemcpyHostToDevice, st));
    { k_diag_q<<<nblk(pr->n_pairs, 128), 128, 0, st>>>(s->basis, pr->n_pairs, pr->pi, pr->pj, pr->ppoff,
                                                     pr->pp, lt.leaf_of_shell, lt.lslo, lt.lshi, nl,
                                                     pr->leaf_base, pr->q); note_launch(); }
    if (pr->n_prim_pairs + pr->n_pairs >= (1ll << 31))
        throw HxfError{HXF_EINVAL, "too many primitive pairs for 32-bit offsets"};
    pr->epp = dalloc<PrimPair>(pr->n_prim_pairs + pr->n_pairs, st);   // + one far-field slot per pair
    pr->eS = dalloc<double>(pr->n_prim_pairs, st);
    pr->fcol = dalloc<uint8_t>(std::max<int64_t>(pr->n_pairs, 1), st);
    {   // HXF_FAR_COLLAPSE=0: every far-field quartet keeps its full primitive lists (A/B hook)
        const char* fc = getenv("HXF_FAR_COLLAPSE");
        const int collapse = fc ? atoi(fc) : 1;
        k_prim_schwarz_sort<<<nblk(pr->n_pairs, 128), 128, 0, st>>>(s->basis, pr->n_pairs, pr->pi, pr->pj, pr->ppoff,
                                                                   pr->pp, pr->epp, pr->eS, pr->n_prim_pairs,
                                                                   collapse, pr->fcol);
        note_launch();
    }
    pr->geo = dalloc<float4>(std::max<int64_t>(pr->n_pairs, 1), st);
    pr->gip = dalloc<float>(std::max<int64_t>(pr->n_pairs, 1), st);
    if (pr->n_pairs) {
        k_pair_geo<<<nblk(pr->n_pairs, 128), 128, 0, st>>>(pr->n_pairs, pr->ppoff, pr->pp, pr->geo, pr->gip);
        note_launch();
    }
    unsigned long long* dsmax = dalloc<unsigned long long>(1, st);
    tmp.push_back(dsmax);
    HXF_CUDA(cudaMemsetAsync(dsmax, 0, sizeof(unsigned long long), st));
    if (pr->n_prim_pairs) { k_maxabs<<<256, 256, 0, st>>>(pr->eS, pr->n_prim_pairs, dsmax); note_launch(); }
    unsigned long long hsm = 0;
    HXF_CUDA(cudaMemcpyAsync(&hsm, dsmax, sizeof(hsm), cudaMemcpyDeviceToHost, st));
    pr->sq = dalloc<double>(pr->n_pairs, st);
    pr->meta = dalloc<uint8_t>(pr->n_pairs, st);
    { k_pair_meta<<<nblk(pr->n_pairs), 256, 0, st>>>(s->basis, pr->n_pairs, pr->pi, pr->pj, pr->q,
                                                     pr->sq, pr->meta); note_launch(); }
    {   // compact ids of the live leaf nodes and their screening vectors
        int* flag = dalloc<int>(nl2 + 1, st);
        tmp.push_back(flag);
        HXF_CUDA(cudaMemsetAsync(flag + nl2, 0, sizeof(int), st));
        { k_live_flags<<<nblk(nl2), 256, 0, st>>>(pr->leaf_base, nl2, flag); note_launch(); }
        pr->ncid = dalloc<int>(nl2 + 1, st);
        size_t tb2 = 0;
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag, pr->ncid, nl2 + 1, st));
        void* tbuf2 = dalloc<char>(tb2, st);
        tmp.push_back(tbuf2);
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(tbuf2, tb2, flag, pr->ncid, nl2 + 1, st));
        int nlive = 0;
        HXF_CUDA(cudaMemcpyAsync(&nlive, pr->ncid + nl2, sizeof(int), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        { k_live_ids<<<nblk(nl2), 256, 0, st>>>(pr->leaf_base, nl2, pr->ncid); note_launch(); }
        pr->nvec = dalloc<double>((int64_t)std::max(nlive, 1) * NVEC, st);
        pr->nvec_tri = dalloc<double>((int64_t)nl * NVEC, st);
        HXF_CUDA(cudaMemsetAsync(pr->nvec_tri, 0, (int64_t)nl * NVEC * sizeof(double), st));
        // the staged leaf screen's node vectors (spans of <= NV_MAXS shells; larger
        // partitions take the unstaged screen, which does not read them)
        if (s->max_leaf_shells <= NV_MAXS)
            { k_node_vectors<<<nblk(nl2, 128), 128, 0, st>>>(lt.lslo, lt.lshi, nl, pr->leaf_base, pr->ncid, pr->q,
                                                           pr->sq, pr->nvec, pr->nvec_tri); note_launch(); }
    }
    double* lnorm = dalloc<double>(nl2, st);
    double* lrow = dalloc<double>(nl2, st);
    double* lcol = dalloc<double>(nl2, st);
    tmp.insert(tmp.end(), {lnorm, lrow, lcol});
    { k_leaf_norms<<<nblk(nl2, 128), 128, 0, st>>>(lt.lslo, lt.lshi, nl, pr->leaf_base, pr->q, lnorm, lrow, lcol); note_launch(); }
    const int64_t nn = s->node_off.back();
    pr->norm = dalloc<double>(nn, st);
    pr->rowsum = dalloc<double>(nn, st);
    pr->colsum = dalloc<double>(nn, st);
    pr->smax = dalloc<double>(nn, st);
    int64_t* d_node_off = dalloc<int64_t>(s->node_off.size(), st);
    tmp.push_back(d_node_off);
    HXF_CUDA(cudaMemcpyAsync(d_node_off, s->node_off.data(), s->node_off.size() * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
    int* d_off = const_cast<int*>(s->lv.off);
    for (int L = s->n_levels - 1; L >= 0; --L) {
        const int n = s->h_off[L + 1] - s->h_off[L];
        const int nnext = L + 1 < s->n_levels ? s->h_off[L + 2] - s->h_off[L + 1] : 0;
        { k_pair_level<<<nblk((int64_t)n * n), 256, 0, st>>>(
            L, n, nnext, d_off + L, s->lv.leaf_id, s->lv.kid0, s->lv.kid1, nl, lnorm, lrow, lcol,
            lsmax, pr->tau_ovlp, d_node_off, pr->norm, pr->rowsum, pr->colsum, pr->smax); note_launch(); }
    }
    // overlap-stage ties: nodes whose block max |S| lies within 1e-12 (relative) of
    // tau_ovlp, the comparison that decides pruning at every level
    if (pr->tau_ovlp > 0.0) {
        const long long cap = 4096;
        TieLog tl{dalloc<hxf_tie_record>(cap, st), dalloc<unsigned long long>(1, st), cap};
        tmp.push_back(tl.rec);
        tmp.push_back(tl.count);
        HXF_CUDA(cudaMemsetAsync(tl.count, 0, sizeof(unsigned long long), st));
        for (int L = 0; L < s->n_levels; ++L) {
            const int n = s->h_off[L + 1] - s->h_off[L];
            k_overlap_ties<<<nblk((int64_t)n * n), 256, 0, st>>>(pr->smax + s->node_off[L], n, L, pr->tau_ovlp, tl);
            note_launch();
        }
        unsigned long long nt = 0;
        HXF_CUDA(cudaMemcpyAsync(&nt, tl.count, sizeof(nt), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        pr->n_ovlp_ties = (int64_t)nt;
        pr->ovlp_ties.resize((size_t)std::min<long long>((long long)nt, cap));
        if (!pr->ovlp_ties.empty()) {
            HXF_CUDA(cudaMemcpyAsync(pr->ovlp_ties.data(), tl.rec, pr->ovlp_ties.size() * sizeof(hxf_tie_record),
                                     cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaStreamSynchronize(st));
        }
    }
    // the traversal's per-node square roots, once per pair tree (correctly rounded:
    // bitwise what a per-visit sqrt would give)
    pr->snorm = dalloc<double>(nn, st);
    pr->srow = dalloc<double>(nn, st);
    pr->scol = dalloc<double>(nn, st);
    { k_node_sqrts<<<nblk(nn), 256, 0, st>>>(nn, pr->norm, pr->rowsum, pr->colsum, pr->snorm, pr->srow, pr->scol); note_launch(); }
    unsigned long long* dmax = dalloc<unsigned long long>(1, st);
    tmp.push_back(dmax);
    HXF_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
    if (pr->n_pairs) { k_maxabs<<<256, 256, 0, st>>>(pr->q, pr->n_pairs, dmax); note_launch(); }
    // K scale bound A(s) = sum over pairs touching shell s of n_f(partner) sqrt(Q)
    double* asum = dalloc<double>(s->ns, st);
    unsigned long long* damax = dalloc<unsigned long long>(1, st);
    tmp.push_back(asum);
    tmp.push_back(damax);
    HXF_CUDA(cudaMemsetAsync(asum, 0, s->ns * sizeof(double), st));
    HXF_CUDA(cudaMemsetAsync(damax, 0, sizeof(unsigned long long), st));
    if (pr->n_pairs) { k_pair_asum<<<nblk(pr->n_pairs), 256, 0, st>>>(s->basis, pr->n_pairs, pr->pi, pr->pj, pr->sq, asum); note_launch(); }
    { k_maxabs<<<64, 256, 0, st>>>(asum, s->ns, damax); note_launch(); }
    unsigned long long ham = 0;
    HXF_CUDA(cudaMemcpyAsync(&ham, damax, sizeof(ham), cudaMemcpyDeviceToHost, st));
    unsigned long long hm = 0;
    HXF_CUDA(cudaMemcpyAsync(&hm, dmax, sizeof(hm), cudaMemcpyDeviceToHost, st));
    for (void* p : tmp) cudaFreeAsync(p, st);
    HXF_CUDA(cudaStreamSynchronize(st));
    HXF_CUDA(cudaGetLastError());
    double mq;
    memcpy(&mq, &hm, sizeof(mq));
    pr->maxq = mq;
    double am;
    memcpy(&am, &ham, sizeof(am));
    pr->amax = am * (1.0 + 1e-12);  // float atomics: the sum is an upper bound up to rounding
    memcpy(&pr->smax_prim, &hsm, sizeof(double));
    int hasp = 0;
    for (int v : s->h_l) hasp |= v;
    pr->has_p = hasp;
}

void trees_build_density(hxf_density* d, const double* P, int on_device, cudaStream_t st) {
    NvtxRange nvtx_range("hxf: density tree");
    hxf_system* s = d->sys;
    std::vector<void*> tmp;
    const int nl = s->n_leaves;
    const int64_t nl2 = (int64_t)nl * nl;
    const int64_t n2 = (int64_t)s->nfn * s->nfn;
    d->P = dalloc<double>(n2, st);
    if (on_device) HXF_CUDA(cudaMemcpyAsync(d->P, P, n2 * sizeof(double), cudaMemcpyDeviceToDevice, st));
    else xfer_to_device(d->P, P, n2 * sizeof(double), st);
    LeafTables lt = make_leaf_tables(s, st, tmp);
    double* lnorm = dalloc<double>(nl2, st);
    tmp.push_back(lnorm);
    { k_density_leaves<<<nblk(nl2, 128), 128, 0, st>>>(d->P, s->nfn, lt.lflo, lt.lfhi, nl, d->zero_drop, lnorm); note_launch(); }
    const int64_t nn = s->node_off.back();
    d->norm = dalloc<double>(nn, st);
    int64_t* d_node_off = dalloc<int64_t>(s->node_off.size(), st);
    tmp.push_back(d_node_off);
    HXF_CUDA(cudaMemcpyAsync(d_node_off, s->node_off.data(), s->node_off.size() * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st));
    int* d_off = const_cast<int*>(s->lv.off);
    for (int L = s->n_levels - 1; L >= 0; --L) {
        const int n = s->h_off[L + 1] - s->h_off[L];
        const int nnext = L + 1 < s->n_levels ? s->h_off[L + 2] - s->h_off[L + 1] : 0;
        { k_density_level<<<nblk((int64_t)n * n), 256, 0, st>>>(L, n, nnext, d_off + L, s->lv.leaf_id,
                                                              s->lv.kid0, s->lv.kid1, nl, lnorm,
                                                              d_node_off, d->norm); note_launch(); }
    }
    unsigned long long* dmax = dalloc<unsigned long long>(1, st);
    tmp.push_back(dmax);
    HXF_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
    { k_maxabs<<<256, 256, 0, st>>>(d->P, n2, dmax); note_launch(); }
    d->pmax = dalloc<double>((int64_t)s->ns * s->ns, st);
    { k_shell_pmax<<<nblk((int64_t)s->ns * s->ns), 256, 0, st>>>(s->basis, d->P, d->pmax); note_launch(); }
    unsigned long long hm = 0;
    HXF_CUDA(cudaMemcpyAsync(&hm, dmax, sizeof(hm), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaMemcpyAsync(&d->frob, d->norm, sizeof(double), cudaMemcpyDeviceToHost, st));
    for (void* p : tmp) cudaFreeAsync(p, st);
    HXF_CUDA(cudaStreamSynchronize(st));
    HXF_CUDA(cudaGetLastError());
    memcpy(&d->maxabs, &hm, sizeof(double));
}
