/*
 * TEST INFRASTRUCTURE ONLY -- never linked into or called by the product path.
 *
 * Streamed CPU restatement of the direct-SCF screening rule of the reference,
 * `dense_exchange_screened` (hexfock/oracle.py:69-108): a shell quartet
 * (i,j,k,l) is evaluated iff
 *
 *     (f(Q_ij) * |P|_jk) * f(Q_kl)  >  tau_2e                (oracle.py:92-96)
 *
 * with f = sqrt (schwarz) or identity (literal) (exchange_naive.py:83-88),
 * Q in canonical orientation (oracle.py:86-90), the same association as the
 * drivers' leaf test (exchange_naive.py:172-182), every product one IEEE
 * binary64 rounding (no FMA: compiled with -ffp-contract=off).  For p shells
 * |P|_jk is the max |P| over the j x k function block.
 *
 * the reference cannot run configs 4-5, so full-size
 * parity of the evaluated set is checked through an order-independent digest
 * (count, sum h(q), sum h(h(q))) mod 2^64, h = SplitMix64 finaliser of
 * ((i*ns + j)*ns + k)*ns + l -- the same digest the device computes
 * (include/hxf.h, hxf_exchange_opts.digest).
 *
 *   naive     : ordered tuples (i,j,k,l) passing the rule (the naive
 *               driver's quartet_log, exchange_naive.py:193-197)
 *   fourfold  : canonical tuples (min(i,j), max(i,j), min(k,l), max(k,l)) of
 *               the naive set -- the four-fold driver's quartet_log
 *               (exchange_symmetry.py:332-340; checked against the Python
 *               oracle in tests/test_direct_digest.py)
 *   eightfold : (fourfold == 2) the fourfold tuples with (i,j) <= (k,l)
 *               lexicographically -- the fourfold set folded bra <-> ket,
 *               the set the optional 8-fold driver evaluates (SURVEY.md 8(a)
 *               S8); the device digest orients each quartet the same way
 *
 * Sampling: only tuples whose first index i satisfies i % mod == rem.
 *
 * Enumeration: per bra pair (a,b), ket rows k in descending |P|_bk order
 * and ket columns l in descending f(Q_kl) order, stopping when the rounded
 * product can no longer exceed tau (binary64 multiplication is monotone).
 *
 * Build: oracle/Makefile -> oracle/libdirect_digest.so (ctypes).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct {
    int ns;
    const double* fq;   /* ns*ns, f(Q), 0 where absent */
    const double* pm;   /* ns*ns, |P| block max */
    const int64_t* qo;  /* row offsets of the sorted f(Q) lists */
    const int32_t* qc;
    const int64_t* po;  /* row offsets of the sorted |P| lists */
    const int32_t* pc;
    double tau, fqmax;
    int fourfold, mod, rem;
    int64_t next;       /* work counter (bra first index), under lock */
    pthread_mutex_t lock;
    uint64_t out[3];
} job_t;

static inline int passes(const job_t* J, int a, int b, int k, int l) {
    const double x = J->fq[(int64_t)a * J->ns + b] * J->pm[(int64_t)b * J->ns + k];
    return x * J->fq[(int64_t)k * J->ns + l] > J->tau;
}

static void* worker(void* arg) {
    job_t* J = (job_t*)arg;
    const int ns = J->ns;
    uint64_t c = 0, h1 = 0, h2 = 0;
    for (;;) {
        pthread_mutex_lock(&J->lock);
        const int64_t a = J->next++;
        pthread_mutex_unlock(&J->lock);
        if (a >= ns) break;
        if (!J->fourfold && J->mod > 1 && a % J->mod != J->rem) continue;
        const int eight = J->fourfold == 2;
        for (int64_t qb = J->qo[a]; qb < J->qo[a + 1]; ++qb) {
            const int b = J->qc[qb];
            if (J->fourfold == 1 && J->mod > 1 && (a < b ? a : b) % J->mod != J->rem) continue;
            const double fab = J->fq[a * (int64_t)ns + b];
            for (int64_t pk = J->po[b]; pk < J->po[b + 1]; ++pk) {
                const int k = J->pc[pk];
                const double x = fab * J->pm[(int64_t)b * ns + k];
                if (x * J->fqmax <= J->tau) break;
                for (int64_t ql = J->qo[k]; ql < J->qo[k + 1]; ++ql) {
                    const int l = J->qc[ql];
                    if (!(x * J->fq[(int64_t)k * ns + l] > J->tau)) break;
                    uint64_t i = a, j = b, kk = k, ll = l;
                    if (J->fourfold) {
                        /* count the canonical tuple once: from the first of
                           its distinct orientations (bra swap bit 1, ket swap
                           bit 0) that passes */
                        const int ci = a < b ? a : b, cj = a < b ? b : a;
                        const int ck = k < l ? k : l, cl = k < l ? l : k;
                        const int o = ((a > b) << 1) | (k > l);
                        int first = 1;
                        for (int o2 = 0; o2 < o && first; ++o2) {
                            if ((o2 & 2) && ci == cj) continue;
                            if ((o2 & 1) && ck == cl) continue;
                            const int a2 = (o2 & 2) ? cj : ci, b2 = (o2 & 2) ? ci : cj;
                            const int k2 = (o2 & 1) ? cl : ck, l2 = (o2 & 1) ? ck : cl;
                            if (passes(J, a2, b2, k2, l2)) first = 0;
                        }
                        if (!first) continue;
                        i = ci; j = cj; kk = ck; ll = cl;
                        if (eight) {
                            if (ci > ck || (ci == ck && cj > cl)) continue;
                            if (J->mod > 1 && (int)(i % (uint64_t)J->mod) != J->rem) continue;
                        }
                    }
                    const uint64_t h = mix64(((i * ns + j) * ns + kk) * ns + ll);
                    c += 1;
                    h1 += h;
                    h2 += mix64(h);
                }
            }
        }
    }
    pthread_mutex_lock(&J->lock);
    J->out[0] += c;
    J->out[1] += h1;
    J->out[2] += h2;
    pthread_mutex_unlock(&J->lock);
    return NULL;
}

typedef struct { double v; int32_t c; } ent_t;

static int cmp_desc(const void* x, const void* y) {
    const ent_t* a = (const ent_t*)x;
    const ent_t* b = (const ent_t*)y;
    if (a->v > b->v) return -1;
    if (a->v < b->v) return 1;
    return a->c - b->c;
}

/* rows of m (ns*ns) with entries > thr, sorted by value descending */
static int sorted_rows(int ns, const double* m, double thr, int64_t** off, int32_t** col) {
    int64_t* o = (int64_t*)malloc(sizeof(int64_t) * (ns + 1));
    if (!o) return -1;
    o[0] = 0;
    for (int r = 0; r < ns; ++r) {
        int64_t n = 0;
        for (int c = 0; c < ns; ++c) n += m[(int64_t)r * ns + c] > thr;
        o[r + 1] = o[r] + n;
    }
    int32_t* cc = (int32_t*)malloc(sizeof(int32_t) * (o[ns] > 0 ? o[ns] : 1));
    ent_t* tmp = (ent_t*)malloc(sizeof(ent_t) * (ns > 0 ? ns : 1));
    if (!cc || !tmp) { free(o); free(cc); free(tmp); return -1; }
    for (int r = 0; r < ns; ++r) {
        int64_t n = 0;
        for (int c = 0; c < ns; ++c) {
            const double v = m[(int64_t)r * ns + c];
            if (v > thr) { tmp[n].v = v; tmp[n].c = c; ++n; }
        }
        qsort(tmp, (size_t)n, sizeof(ent_t), cmp_desc);
        for (int64_t t = 0; t < n; ++t) cc[o[r] + t] = tmp[t].c;
    }
    free(tmp);
    *off = o;
    *col = cc;
    return 0;
}

/*
 * q: ns*ns shell-pair Q (canonical orientation, symmetric; < 0 or 0 = absent)
 * pmax: ns*ns block max |P|
 * mode: 0 schwarz (f = sqrt), 1 literal
 * returns 0 on success, out = {count, sum h, sum h(h)}
 */
int direct_digest(int ns, const double* q, const double* pmax, double tau, int mode, int fourfold,
                  int mod, int rem, int nthreads, uint64_t* out) {
    const int64_t n2 = (int64_t)ns * ns;
    double* fq = (double*)malloc(sizeof(double) * (n2 > 0 ? n2 : 1));
    if (!fq) return -1;
    double fqmax = 0.0;
    for (int64_t t = 0; t < n2; ++t) {
        const double v = q[t] > 0.0 ? (mode == 0 ? sqrt(q[t]) : q[t]) : 0.0;
        fq[t] = v;
        if (v > fqmax) fqmax = v;
    }
    int64_t *qo = NULL, *po = NULL;
    int32_t *qc = NULL, *pc = NULL;
    /* an entry can only matter if it is non-zero; the loops stop by value */
    if (sorted_rows(ns, fq, 0.0, &qo, &qc) || sorted_rows(ns, pmax, 0.0, &po, &pc)) {
        free(fq); free(qo); free(qc); free(po); free(pc);
        return -1;
    }
    job_t J;
    memset(&J, 0, sizeof(J));
    J.ns = ns; J.fq = fq; J.pm = pmax; J.qo = qo; J.qc = qc; J.po = po; J.pc = pc;
    J.tau = tau; J.fqmax = fqmax; J.fourfold = fourfold; J.mod = mod; J.rem = rem;
    pthread_mutex_init(&J.lock, NULL);
    if (nthreads < 1) nthreads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * nthreads);
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
        if (pthread_create(&th[t], NULL, worker, &J) == 0) ++started;
    if (started == 0) worker(&J);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    pthread_mutex_destroy(&J.lock);
    free(th);
    out[0] = J.out[0];
    out[1] = J.out[1];
    out[2] = J.out[2];
    free(fq); free(qo); free(qc); free(po); free(pc);
    return 0;
}
