/*
 * TEST INFRASTRUCTURE ONLY -- never linked into or called by the product path.
 *
 * Independent CPU restatement of the pieces a full-size parity check needs
 * ("for K, use the same restatement on a sampled set
 * of K rows"), written without any of the device code:
 *
 *   kref_q     overlap pruning of leaf pair blocks (quadtree.py:298-301 with
 *              the contracted overlap of integrals.py:58-64; p shells use the
 *              s-proxy overlap of their primitives) and the canonical
 *              Schwarz diagonal Q_ij = max_f (i_f j_f|i_f j_f) over present
 *              pairs (integrals.py:219-222, quadtree.py:307-313); 0 = absent.
 *   kref_rows  rows of the naive exchange K over the direct-SCF keep set
 *              (oracle.py:69-108): quartet (i,j,k,l) kept iff
 *              (f(Q_ij) |P|_jk) f(Q_kl) > tau, contributing
 *              K[i_x, l_w] += -1/2 P[j_y, k_z] (i_x j_y|k_z l_w)
 *              (exchange_naive.py:185-192).  The fourfold / eightfold K is
 *              the symmetrised naive K, so its rows are compared against
 *              these too.
 *
 * ERIs: contracted Cartesian s/p shells by the Obara-Saika vertical
 * recursion onto [e0|f0]^(m) per primitive quartet, summed over primitives,
 * then the Head-Gordon-Pople horizontal transfer -- the textbook scheme the
 * Python oracle (oracle/hexfock_oracle.py:eri_general) states, restated here
 * as a generic table-driven recursion (no generated code).  Boys F_m:
 * the reference's series below t = 12 (integrals.py:40-50, extended to
 * F_m by the downward recursion) and erf + upward recursion above
 * (integrals.py:51-54).  Everything is plain binary64 (-ffp-contract=off).
 *
 * Build: oracle/Makefile -> oracle/libkref.so (ctypes front end oracle/kref.py).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define LMAX 1            /* per shell */
#define EMAX (2 * LMAX)   /* la + lb */
#define MMAX (4 * LMAX)   /* la + lb + lc + ld */
#define NCART_UPTO 10     /* Cartesian monomials with |e| <= 2 */

/* ------------------------------------------------------------------ */
/* Cartesian monomials with |e| <= 2: index 0 = 1, 1-3 = x y z, 4-9 = xx xy xz yy yz zz */
static const int CART[NCART_UPTO][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {2, 0, 0},
                                         {1, 1, 0}, {1, 0, 1}, {0, 2, 0}, {0, 1, 1}, {0, 0, 2}};

static int cart_index(int x, int y, int z) {
    for (int t = 0; t < NCART_UPTO; ++t)
        if (CART[t][0] == x && CART[t][1] == y && CART[t][2] == z) return t;
    return -1;
}

static int ncart_upto(int l) { return l == 0 ? 1 : (l == 1 ? 4 : 10); }
static int cart_lo(int l) { return l == 0 ? 0 : (l == 1 ? 1 : 4); }

/* e - 1_i and e + 1_i lookups */
static int SUB1[NCART_UPTO][3], ADD1[NCART_UPTO][3];

static void init_tables(void) {
    static int done = 0;
    if (done) return;
    for (int t = 0; t < NCART_UPTO; ++t)
        for (int i = 0; i < 3; ++i) {
            int e[3] = {CART[t][0], CART[t][1], CART[t][2]};
            if (e[i] > 0) {
                e[i]--;
                SUB1[t][i] = cart_index(e[0], e[1], e[2]);
                e[i]++;
            } else {
                SUB1[t][i] = -1;
            }
            e[i]++;
            ADD1[t][i] = (e[0] + e[1] + e[2] <= 2) ? cart_index(e[0], e[1], e[2]) : -1;
        }
    done = 1;
}

/* ------------------------------------------------------------------ */
/* Boys F_m(t), m = 0..mmax */
static void boys(double t, int mmax, double* F) {
    if (t < 12.0) {
        /* F_mmax = e^{-t} sum_k (2t)^k / ((2m+1)(2m+3)...(2m+2k+1)) */
        const double et = exp(-t);
        double term = 1.0 / (2 * mmax + 1), sum = term;
        for (int k = 1; k < 200; ++k) {
            term *= 2.0 * t / (2 * mmax + 2 * k + 1);
            sum += term;
            if (term < 1e-18 * sum) break;
        }
        F[mmax] = et * sum;
        for (int m = mmax; m > 0; --m) F[m - 1] = (2.0 * t * F[m] + et) / (2 * m - 1);
    } else {
        const double st = sqrt(t);
        F[0] = 0.5 * sqrt(M_PI / t) * erf(st);
        const double et = exp(-t);
        for (int m = 0; m < mmax; ++m) F[m + 1] = ((2 * m + 1) * F[m] - et) / (2.0 * t);
    }
}

/* ------------------------------------------------------------------ */
typedef struct {
    int ns, nfn;
    const double* ctr;   /* ns x 3 */
    const int* l;        /* ns */
    const int* poff;     /* ns + 1 */
    const double* ex;    /* exponents */
    const double* w;     /* normalised primitive weights (l-specific) */
    const double* sw;    /* s-proxy weights (overlap pruning) */
    const int* fn;       /* ns, first function */
} basis_t;

static int nfun(int l) { return l == 0 ? 1 : 3; }

/* Contracted block (ij|kl), out[((x*nj+y)*nk+z)*nl+w], Cartesian p order x y z. */
static void eri_block(const basis_t* b, int si, int sj, int sk, int sl, double* out) {
    const int la = b->l[si], lb = b->l[sj], lc = b->l[sk], ld = b->l[sl];
    const int L = la + lb + lc + ld, le = la + lb, lf = lc + ld;
    const double* A = b->ctr + 3 * si;
    const double* B = b->ctr + 3 * sj;
    const double* C = b->ctr + 3 * sk;
    const double* D = b->ctr + 3 * sl;
    const int ne = ncart_upto(le), nf = ncart_upto(lf);
    /* contracted [e0|f0], e, f indices < ne, nf */
    double E[NCART_UPTO][NCART_UPTO];
    memset(E, 0, sizeof(E));
    double AB2 = 0.0, CD2 = 0.0;
    for (int i = 0; i < 3; ++i) {
        AB2 += (A[i] - B[i]) * (A[i] - B[i]);
        CD2 += (C[i] - D[i]) * (C[i] - D[i]);
    }
    /* V[m][e][f] scratch */
    double V[MMAX + 1][NCART_UPTO][NCART_UPTO];
    for (int pa = b->poff[si]; pa < b->poff[si + 1]; ++pa)
        for (int pb = b->poff[sj]; pb < b->poff[sj + 1]; ++pb) {
            const double a = b->ex[pa], bb = b->ex[pb], p = a + bb;
            const double Kab = b->w[pa] * b->w[pb] * exp(-a * bb / p * AB2);
            double Pc[3];
            for (int i = 0; i < 3; ++i) Pc[i] = (a * A[i] + bb * B[i]) / p;
            for (int pc = b->poff[sk]; pc < b->poff[sk + 1]; ++pc)
                for (int pd = b->poff[sl]; pd < b->poff[sl + 1]; ++pd) {
                    const double c = b->ex[pc], d = b->ex[pd], q = c + d;
                    const double Kcd = b->w[pc] * b->w[pd] * exp(-c * d / q * CD2);
                    double Qc[3], W[3], PQ2 = 0.0;
                    for (int i = 0; i < 3; ++i) {
                        Qc[i] = (c * C[i] + d * D[i]) / q;
                        W[i] = (p * Pc[i] + q * Qc[i]) / (p + q);
                        PQ2 += (Pc[i] - Qc[i]) * (Pc[i] - Qc[i]);
                    }
                    const double rho = p * q / (p + q);
                    const double pref = 2.0 * pow(M_PI, 2.5) / (p * q * sqrt(p + q)) * Kab * Kcd;
                    double F[MMAX + 1];
                    boys(rho * PQ2, L, F);
                    /* [0|0]^(m) */
                    for (int m = 0; m <= L; ++m) V[m][0][0] = pref * F[m];
                    /* build e up to le with f = 0 (orders m <= L - |e|) */
                    for (int e = 1; e < ne; ++e) {
                        const int ln = CART[e][0] + CART[e][1] + CART[e][2];
                        int i = 0;
                        while (SUB1[e][i] < 0) ++i;
                        const int e1 = SUB1[e][i];
                        const int e2 = SUB1[e1][i];
                        const int n1 = CART[e1][i];
                        for (int m = 0; m <= L - ln; ++m) {
                            double v = (Pc[i] - A[i]) * V[m][e1][0] + (W[i] - Pc[i]) * V[m + 1][e1][0];
                            if (e2 >= 0) v += n1 / (2.0 * p) * (V[m][e2][0] - rho / p * V[m + 1][e2][0]);
                            V[m][e][0] = v;
                        }
                    }
                    /* then f up to lf for every e */
                    for (int f = 1; f < nf; ++f) {
                        const int lnf = CART[f][0] + CART[f][1] + CART[f][2];
                        int i = 0;
                        while (SUB1[f][i] < 0) ++i;
                        const int f1 = SUB1[f][i];
                        const int f2 = SUB1[f1][i];
                        const int n1 = CART[f1][i];
                        for (int e = 0; e < ne; ++e) {
                            const int lne = CART[e][0] + CART[e][1] + CART[e][2];
                            const int em = SUB1[e][i];
                            for (int m = 0; m <= L - lne - lnf; ++m) {
                                double v = (Qc[i] - C[i]) * V[m][e][f1] + (W[i] - Qc[i]) * V[m + 1][e][f1];
                                if (f2 >= 0) v += n1 / (2.0 * q) * (V[m][e][f2] - rho / q * V[m + 1][e][f2]);
                                if (em >= 0) v += CART[e][i] / (2.0 * (p + q)) * V[m + 1][em][f1];
                                V[m][e][f] = v;
                            }
                        }
                    }
                    for (int e = cart_lo(la); e < ne; ++e)
                        for (int f = cart_lo(lc); f < nf; ++f) E[e][f] += V[0][e][f];
                }
        }
    /* horizontal transfer: (a b| = (a+1_i b-1_i| + AB_i (a b-1_i|, lb, ld <= 1 */
    const int ni = nfun(la), nj = nfun(lb), nk = nfun(lc), nl = nfun(ld);
    for (int x = 0; x < ni; ++x)
        for (int y = 0; y < nj; ++y)
            for (int z = 0; z < nk; ++z)
                for (int t = 0; t < nl; ++t) {
                    const int ea = la ? 1 + x : 0, fc = lc ? 1 + z : 0;
                    /* bra: (ea, y| -> [ea+1_y | ...] + AB_y [ea|...] */
                    double v = 0.0;
                    for (int tb = 0; tb < (lb ? 2 : 1); ++tb) {
                        int e;
                        double cb;
                        if (!lb) { e = ea; cb = 1.0; }
                        else if (tb == 0) { e = ADD1[ea][y]; cb = 1.0; }
                        else { e = ea; cb = A[y] - B[y]; }
                        for (int td = 0; td < (ld ? 2 : 1); ++td) {
                            int f;
                            double cd;
                            if (!ld) { f = fc; cd = 1.0; }
                            else if (td == 0) { f = ADD1[fc][t]; cd = 1.0; }
                            else { f = fc; cd = C[t] - D[t]; }
                            v += cb * cd * E[e][f];
                        }
                    }
                    out[((x * nj + y) * nk + z) * nl + t] = v;
                }
}

/* exported for the CPU tests: one contracted block */
int kref_eri_block(int ns, const double* ctr, const int* l, const int* poff, const double* ex, const double* w,
                   int si, int sj, int sk, int sl, double* out) {
    init_tables();
    basis_t b = {ns, 0, ctr, l, poff, ex, w, NULL, NULL};
    for (int s = 0; s < ns; ++s)
        if (l[s] < 0 || l[s] > LMAX) return 1;
    eri_block(&b, si, sj, sk, sl, out);
    return 0;
}

/* ------------------------------------------------------------------ */
/* overlap pruning + Q */

static double overlap_s(const basis_t* b, int i, int j) {
    double r2 = 0.0;
    for (int t = 0; t < 3; ++t) {
        const double d = b->ctr[3 * i + t] - b->ctr[3 * j + t];
        r2 += d * d;
    }
    double s = 0.0;
    for (int pa = b->poff[i]; pa < b->poff[i + 1]; ++pa)
        for (int pb = b->poff[j]; pb < b->poff[j + 1]; ++pb) {
            const double a = b->ex[pa], c = b->ex[pb], p = a + c;
            s += b->sw[pa] * b->sw[pb] * pow(M_PI / p, 1.5) * exp(-a * c / p * r2);
        }
    return s;
}

typedef struct {
    const basis_t* b;
    int nleaf;
    const int* lslo;
    const int* lshi;
    const double* lc;    /* leaf centroid x3 */
    const double* lr;    /* leaf radius */
    double tau_ovlp, spref, mu_min;
    double* q;           /* ns x ns */
    int64_t next;
    pthread_mutex_t lock;
} qjob_t;

static void* q_worker(void* arg) {
    qjob_t* J = (qjob_t*)arg;
    const basis_t* b = J->b;
    const int ns = b->ns;
    double blk[81];
    for (;;) {
        pthread_mutex_lock(&J->lock);
        const int64_t A = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (A >= J->nleaf) break;
        for (int Bl = 0; Bl < J->nleaf; ++Bl) {
            /* rigorous skip: every |S_ij| <= spref exp(-mu_min d^2) with d the
               distance between the leaves' bounding spheres */
            double dc = 0.0;
            for (int t = 0; t < 3; ++t) {
                const double d = J->lc[3 * A + t] - J->lc[3 * Bl + t];
                dc += d * d;
            }
            double d = sqrt(dc) - J->lr[A] - J->lr[Bl];
            if (d > 0.0 && J->spref * exp(-J->mu_min * d * d) < 0.5 * J->tau_ovlp) continue;
            double smax = 0.0;
            for (int i = J->lslo[A]; i < J->lshi[A]; ++i)
                for (int j = J->lslo[Bl]; j < J->lshi[Bl]; ++j) {
                    const double s = fabs(overlap_s(b, i, j));
                    if (s > smax) smax = s;
                }
            if (smax < J->tau_ovlp) continue;   /* pruned leaf block (quadtree.py:298-301) */
            for (int i = J->lslo[A]; i < J->lshi[A]; ++i)
                for (int j = J->lslo[Bl]; j < J->lshi[Bl]; ++j) {
                    const int ci = i < j ? i : j, cj = i < j ? j : i;
                    eri_block(b, ci, cj, ci, cj, blk);
                    const int ni = nfun(b->l[ci]), nj = nfun(b->l[cj]);
                    double m = blk[0];
                    for (int x = 0; x < ni; ++x)
                        for (int y = 0; y < nj; ++y) {
                            const double v = blk[((x * nj + y) * ni + x) * nj + y];
                            if (v > m) m = v;
                        }
                    J->q[(int64_t)i * ns + j] = m;
                }
        }
    }
    return NULL;
}

int kref_q(int ns, const double* ctr, const int* l, const int* poff, const double* ex, const double* w,
           const double* sw, int nleaf, const int* lslo, const int* lshi, double tau_ovlp, int threads,
           double* q) {
    init_tables();
    basis_t b = {ns, 0, ctr, l, poff, ex, w, sw, NULL};
    memset(q, 0, sizeof(double) * (size_t)ns * ns);
    double* lc = (double*)calloc((size_t)nleaf * 3, sizeof(double));
    double* lr = (double*)calloc((size_t)nleaf, sizeof(double));
    if (!lc || !lr) return 1;
    for (int A = 0; A < nleaf; ++A) {
        const int n = lshi[A] - lslo[A];
        for (int i = lslo[A]; i < lshi[A]; ++i)
            for (int t = 0; t < 3; ++t) lc[3 * A + t] += ctr[3 * i + t] / n;
        double r = 0.0;
        for (int i = lslo[A]; i < lshi[A]; ++i) {
            double d2 = 0.0;
            for (int t = 0; t < 3; ++t) d2 += (ctr[3 * i + t] - lc[3 * A + t]) * (ctr[3 * i + t] - lc[3 * A + t]);
            if (sqrt(d2) > r) r = sqrt(d2);
        }
        lr[A] = r * (1.0 + 1e-12) + 1e-12;
    }
    /* spref = max_ij sum_ab |sw_a sw_b| (pi/p)^1.5 (upper bound ignoring the
       Gaussian factor); mu_min = min_ab ab/(a+b) */
    double mu_min = INFINITY, wmax = 0.0, emin = INFINITY;
    int kmax = 0;
    for (int s = 0; s < ns; ++s) {
        const int k = poff[s + 1] - poff[s];
        if (k > kmax) kmax = k;
        for (int p = poff[s]; p < poff[s + 1]; ++p) {
            if (fabs(sw[p]) > wmax) wmax = fabs(sw[p]);
            if (ex[p] < emin) emin = ex[p];
        }
    }
    for (int s = 0; s < ns; ++s)
        for (int p = poff[s]; p < poff[s + 1]; ++p) {
            const double mu = ex[p] * emin / (ex[p] + emin);   /* ab/(a+b) is increasing in each */
            if (mu < mu_min) mu_min = mu;
        }
    const double spref = (double)kmax * kmax * wmax * wmax * pow(M_PI / (2.0 * emin), 1.5);
    qjob_t J;
    J.b = &b;
    J.nleaf = nleaf;
    J.lslo = lslo;
    J.lshi = lshi;
    J.lc = lc;
    J.lr = lr;
    J.tau_ovlp = tau_ovlp;
    J.spref = tau_ovlp > 0.0 ? spref : INFINITY;
    J.mu_min = mu_min;
    J.q = q;
    J.next = 0;
    pthread_mutex_init(&J.lock, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, q_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.lock);
    free(lc);
    free(lr);
    return 0;
}

/* ------------------------------------------------------------------ */
/* K rows */

typedef struct {
    const basis_t* b;
    const double* q;     /* ns x ns canonical Q, <= 0 absent */
    const double* P;     /* nfn x nfn */
    double tau;
    int mode;
    const int* rows;     /* shell ids */
    int nrows;
    const int64_t* ro;   /* per row shell i: sorted present partners */
    const int32_t* rc;
    double fqmax;
    double* out;         /* (sum nfun(rows)) x nfn */
    const int* outoff;   /* row offset per requested shell */
    int64_t next;        /* work item = (row r, partner index) */
    int64_t nwork;
    const int64_t* wo;   /* work offsets per requested row */
    pthread_mutex_t lock;
    long long nq;
} rjob_t;

static double fqv(const rjob_t* J, int a, int c) {
    const int ns = J->b->ns;
    const double v = J->q[(int64_t)a * ns + c];
    if (v <= 0.0) return 0.0;
    return J->mode == 0 ? sqrt(v) : v;
}

static double pmaxblk(const rjob_t* J, int j, int k) {
    const basis_t* b = J->b;
    double m = 0.0;
    for (int y = 0; y < nfun(b->l[j]); ++y)
        for (int z = 0; z < nfun(b->l[k]); ++z) {
            const double v = fabs(J->P[(int64_t)(b->fn[j] + y) * b->nfn + b->fn[k] + z]);
            if (v > m) m = v;
        }
    return m;
}

static void* r_worker(void* arg) {
    rjob_t* J = (rjob_t*)arg;
    const basis_t* b = J->b;
    const int ns = b->ns, nfn = b->nfn;
    double blk[81];
    double* acc = (double*)calloc((size_t)3 * nfn, sizeof(double));
    long long nq = 0;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        const int64_t it = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (it >= J->nwork) break;
        int r = 0;
        while (J->wo[r + 1] <= it) ++r;
        const int i = J->rows[r];
        const int j = J->rc[J->ro[i] + (it - J->wo[r])];
        const double fij = fqv(J, i < j ? i : j, i < j ? j : i);
        if (fij <= 0.0) continue;
        const int ni = nfun(b->l[i]), nj = nfun(b->l[j]);
        memset(acc, 0, sizeof(double) * 3 * nfn);
        for (int k = 0; k < ns; ++k) {
            const double pm = pmaxblk(J, j, k);
            const double x = fij * pm;
            if (!(x * J->fqmax > J->tau)) continue;
            const int nk = nfun(b->l[k]);
            for (int64_t t = J->ro[k]; t < J->ro[k + 1]; ++t) {
                const int l = J->rc[t];
                const double fkl = fqv(J, k < l ? k : l, k < l ? l : k);
                if (!(x * fkl > J->tau)) continue;
                const int nl = nfun(b->l[l]);
                eri_block(b, i, j, k, l, blk);
                ++nq;
                for (int xx = 0; xx < ni; ++xx)
                    for (int w = 0; w < nl; ++w) {
                        double s = 0.0;
                        for (int y = 0; y < nj; ++y)
                            for (int z = 0; z < nk; ++z)
                                s += J->P[(int64_t)(b->fn[j] + y) * nfn + b->fn[k] + z] *
                                     blk[((xx * nj + y) * nk + z) * nl + w];
                        acc[(int64_t)xx * nfn + b->fn[l] + w] += -0.5 * s;
                    }
            }
        }
        pthread_mutex_lock(&J->lock);
        for (int xx = 0; xx < ni; ++xx) {
            double* o = J->out + (int64_t)(J->outoff[r] + xx) * nfn;
            const double* a = acc + (int64_t)xx * nfn;
            for (int c = 0; c < nfn; ++c) o[c] += a[c];
        }
        pthread_mutex_unlock(&J->lock);
    }
    pthread_mutex_lock(&J->lock);
    J->nq += nq;
    pthread_mutex_unlock(&J->lock);
    free(acc);
    return NULL;
}

/* rows of the naive K for the requested shells; out has sum_r nfun(l[rows[r]])
   rows of nfn doubles (zeroed here).  Returns the number of evaluated shell
   quartets through *nquart. */
int kref_rows(int ns, int nfn, const double* ctr, const int* l, const int* poff, const double* ex,
              const double* w, const int* fn, const double* q, const double* P, double tau, int mode,
              int nrows, const int* rows, int threads, double* out, long long* nquart) {
    init_tables();
    basis_t b = {ns, nfn, ctr, l, poff, ex, w, NULL, fn};
    /* present partners per shell (q > 0 in either orientation) */
    int64_t* ro = (int64_t*)calloc((size_t)ns + 1, sizeof(int64_t));
    if (!ro) return 1;
    double fqmax = 0.0;
    for (int a = 0; a < ns; ++a) {
        int64_t c = 0;
        for (int t = 0; t < ns; ++t) {
            const double v = q[(int64_t)(a < t ? a : t) * ns + (a < t ? t : a)];
            if (v > 0.0) {
                ++c;
                const double f = mode == 0 ? sqrt(v) : v;
                if (f > fqmax) fqmax = f;
            }
        }
        ro[a + 1] = ro[a] + c;
    }
    int32_t* rc = (int32_t*)malloc(sizeof(int32_t) * (size_t)(ro[ns] ? ro[ns] : 1));
    if (!rc) return 1;
    for (int a = 0; a < ns; ++a) {
        int64_t c = ro[a];
        for (int t = 0; t < ns; ++t)
            if (q[(int64_t)(a < t ? a : t) * ns + (a < t ? t : a)] > 0.0) rc[c++] = t;
    }
    int* outoff = (int*)malloc(sizeof(int) * (nrows + 1));
    int64_t* wo = (int64_t*)malloc(sizeof(int64_t) * (nrows + 1));
    outoff[0] = 0;
    wo[0] = 0;
    for (int r = 0; r < nrows; ++r) {
        outoff[r + 1] = outoff[r] + nfun(l[rows[r]]);
        wo[r + 1] = wo[r] + (ro[rows[r] + 1] - ro[rows[r]]);
    }
    memset(out, 0, sizeof(double) * (size_t)outoff[nrows] * nfn);
    rjob_t J;
    J.b = &b;
    J.q = q;
    J.P = P;
    J.tau = tau;
    J.mode = mode;
    J.rows = rows;
    J.nrows = nrows;
    J.ro = ro;
    J.rc = rc;
    J.fqmax = fqmax;
    J.out = out;
    J.outoff = outoff;
    J.next = 0;
    J.nwork = wo[nrows];
    J.wo = wo;
    J.nq = 0;
    pthread_mutex_init(&J.lock, NULL);
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, r_worker, &J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
    pthread_mutex_destroy(&J.lock);
    if (nquart) *nquart = J.nq;
    free(ro);
    free(rc);
    free(outoff);
    free(wo);
    return 0;
}
