// Leaf stage of the exchange build (SURVEY.md kernel K6) and the K epilogue (K7).
//
//   screen   per-quartet Schwarz test of every leaf task, one warp per task
//            (exchange_naive.py:156-182, exchange_symmetry.py:296-331):
//            bound = (f(Q_ij) |P|) f(Q_kl), keep iff bound > tau; counters and
//            the culled-bound ledger; survivors compacted (ballot + warp-
//            aggregated atomics) into a bounded record buffer.
//   sort     survivors bucketed by angular class (4-bit radix pass) so each
//            ERI launch is class-uniform (no divergence between s and p code).
//   eri      Obara-Saika/HGP ERIs (eri_classes.cuh), one thread per shell
//            quartet, contracted into K with the density: naive slot
//            K[i,l] += -1/2 P[j,k] (ij|kl) (exchange_naive.py:191-192); the
//            4-fold scatter of exchange_symmetry.py:345-361 with its
//            diagonal weights.  K accumulates in 64-bit fixed point with
//            integer atomics, so the result is bitwise reproducible.
//   epilogue fixed point -> FP64; fourfold: asymmetry check and (K+K^T)/2
//            (symmetrize_final, exchange_symmetry.py:197-209).
// Leaf tasks are processed in chunks sized so the survivor buffer never
// overflows; chunk boundaries depend only on the data (deterministic).

#include <cub/cub.cuh>

#include <algorithm>
#include <type_traits>
#include <cmath>
#include <cstring>

#include "boys.cuh"
#include "hxf_internal.cuh"
#define boys_eval boys_bf_scaled  // ERI kernels: the short-chain Boys variant
#include "eri_classes.cuh"
#include "traverse.cuh"

#ifndef HXF_ERI_NOFAR   // 1: A/B build without the far-field path (every quartet on the table path)
#define HXF_ERI_NOFAR 0
#endif

#define SCREEN_WARPS 4     // k_screen (any span size)
#define STAGED_MAXS 10     // k_screen2 stages spans of <= 10 shells (NV_MAXS node vectors)

namespace {

struct ScreenArgs {
    const uint64_t* tasks;
    int64_t t0, t1;
    int tblock;               // k_screen2: a warp takes runs of tblock consecutive tasks (block-cyclic)
    unsigned* next_run;       // k_screen2: non-NULL = runs are handed out dynamically (zeroed per launch)
    const int* lslo;
    const int* lshi;
    int nleaf;
    const int64_t* bra_base;
    const int64_t* ket_base;
    const double* qb;
    const double* qk;
    const int* l;
    const int* poff;
    const double* sqb;        // sqrt(Q) per bra / ket pair id
    const double* sqk;
    const uint8_t* metab;     // class bits | primitive count per pair id
    const uint8_t* metak;
    const double* pmax;       // shell-level max |P| (n_shells^2)
    int ns;
    const int* fn;
    const int* nf;
    const double* P;
    int nfn;
    double tau;
    int mode;
    uint64_t* rec;
    uint16_t* keys;
    int64_t cap;
    unsigned long long* fill;
    long long* counters;
    unsigned long long* ledger;
    const int* ncidb;         // bra / ket pair trees: compact live-node ids and node vectors
    const double* nvecb;
    const double* nvecb_tri;
    const int* ncidk;
    const double* nveck;
    const double* nveck_tri;
    const int* bpi;           // shells of the bra / ket pair ids (tie records)
    const int* bpj;
    const int* kpi;
    const int* kpj;
    TieLog ties;
    int64_t n_bpairs, n_kpairs;   // pair table sizes (HXF_DEBUG_BOUNDS checks)
};

// Far field (ERI key bit 12): every primitive quartet of a shell quartet has
// Boys argument T = |P-Q|^2 / (1/p + 1/q) >= boys_far_t(L); decided per shell
// quartet from the two pairs' enclosing spheres (k_pair_geo, k_classify_far).
// Such quartets sort into their own ERI range whose kernels evaluate only the
// asymptotic Boys branch (the branch the table path selects there).
// (An 8-bit key -- far, class, min(nk, 8), one radix pass instead of two -- saves
// ~170 ms of sort per c5 build and costs 880 ms in the ERI kernels, whose warps then mix
// bra primitive counts: profiles/r02_ab_eri_memory.log.  13 bits stay.)
// ERI bin of a survivor (written over the screen's 12-bit class / count key by
// k_binb_classify): ((far * 16 + class) * 9 + nb-1) * 9 + nk-1, 2592 bins (a pair has at most
// 3 x 3 primitives); slab padding goes to bin ERI_NBINS.  One ERI kernel per (far, class)
// reads the 81 bins of its primitive-count combinations as one record range.
// (Measured and dropped: bra pair id bits appended to the key -- with the leaf tasks in
// bra-node-major order 2 / 3 extra bits cost 80 / 106 ms of ERI kernels at c5: they scatter a
// leaf task's run over sub-ranges and lose more ket-side locality than the bra side gains.)
#define ERI_NBINS 2592
#define KEY_CLASS_SPAN 81
#define KEY_OF(far, cls) ((((far) ? 16 : 0) + (cls)) * KEY_CLASS_SPAN)

// Survivor emission through per-warp slabs: one global atomic reserves SLAB
// record slots; a slab that cannot take the next ballot is padded with
// sentinel records (key 0xFFFF sorts after every real 12-bit key and is
// excluded by the key bounds), so no emitting iteration waits for an atomic.
#define SLAB 1024
#define SENTINEL_REC (~0ull)
#define SENTINEL_KEY ((uint16_t)0xFFFF)

struct Slab {
    unsigned long long base;
    int used;
};

// a leaf-stage tie: shell ids from the pair ids (cold path, not inlined)
static __device__ __noinline__ void tie_emit_leaf(TieLog tl, const int* bpi, const int* bpj, const int* kpi, const int* kpj,
                                           int64_t pa, int64_t pk, int slot, double bound, double tau) {
    tie_emit(tl, HXF_TIE_LEAF, -1, slot, bound > tau, bpi[pa], bpj[pa], kpi[pk], kpj[pk], bound, tau);
}

template <typename Args>
__device__ __forceinline__ void slab_pad(const Slab& s, const Args& a, int lane) {
    for (int i = s.used + lane; i < SLAB; i += 32) {
        const unsigned long long pos = s.base + i;
        if ((int64_t)pos < a.cap) {
            a.rec[pos] = SENTINEL_REC;
            a.keys[pos] = SENTINEL_KEY;
        }
    }
}

template <typename Args>
__device__ __forceinline__ void slab_emit(Slab& s, const Args& a, unsigned bal, bool keep, uint64_t rec,
                                          uint16_t key, int lane) {
    const int cnt = __popc(bal);
    if (s.used + cnt > SLAB) {  // warp-uniform
        slab_pad(s, a, lane);
        unsigned long long b = 0;
        if (lane == 0) b = atomicAdd(a.fill, (unsigned long long)SLAB);
        s.base = __shfl_sync(0xffffffffu, b, 0);
        s.used = 0;
    }
    if (keep) {
        const unsigned long long pos = s.base + s.used + __popc(bal & ((1u << lane) - 1u));
        HXF_BCHECK((int64_t)(rec & 0xfffffff) < a.n_bpairs && (int64_t)((rec >> 28) & 0xfffffff) < a.n_kpairs,
                   a.counters);
        if ((int64_t)pos < a.cap) {
            a.rec[pos] = rec;
            a.keys[pos] = key;
        }
    }
    s.used += cnt;
}

// canonical (x <= y) enumeration of a diagonal node's pairs
__device__ __forceinline__ void tri_decode(int a, int n, int* x, int* y) {
    int r = 0;
    while (a >= n - r) {
        a -= n - r;
        ++r;
    }
    *x = r;
    *y = r + a;
}

// Per-quartet leaf screen for any leaf span size (the reference's --leaf-size
// takes any value, cli.py:289): one warp per leaf task, every quartet tested
// from global memory (no per-warp staging, so no bound on the span size).
// The path for partitions whose leaf spans exceed the staged screen's 10
// shells, and the A/B reference of k_screen2 (HXF_SCREEN=flat); same
// decisions, counters and ledger.
// TIES: the diagnostic instantiation that also appends tie records (second pass, run
// only when a build counted leaf ties and the caller asked for the log).
template <bool SYM, bool EMIT, bool EIGHT = false, bool TIES = false>
__global__ void __launch_bounds__(SCREEN_WARPS * 32) k_screen(ScreenArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = blockIdx.x * (int64_t)SCREEN_WARPS + (threadIdx.x >> 5);
    const int64_t W = (int64_t)gridDim.x * SCREEN_WARPS;
    long long n_eri = 0, n_cull = 0, n_tie = 0;
    Slab slab{0ull, SLAB};
    double ledger = 0.0;
    const bool schwarz = a.mode == HXF_MODE_SCHWARZ;
    const double tie_lo = a.tau * (1.0 - 1e-12), tie_hi = a.tau * (1.0 + 1e-12);
    for (int64_t t = a.t0 + gw; t < a.t1; t += W) {
        const uint64_t task = a.tasks[t];
        const int mu = task & 0x7fff, nu = (task >> 15) & 0x7fff, lam = (task >> 30) & 0x7fff,
                  sig = (task >> 45) & 0x7fff;
        const int live = SYM ? (int)(task >> 60) : 1;
        const int smu = a.lslo[mu], snu = a.lslo[nu], slam = a.lslo[lam], ssig = a.lslo[sig];
        const int nmu = a.lshi[mu] - smu, nnu = a.lshi[nu] - snu, nlam = a.lshi[lam] - slam,
                  nsig = a.lshi[sig] - ssig;
        const int64_t bb = a.bra_base[(int64_t)mu * a.nleaf + nu];
        const int64_t kb = a.ket_base[(int64_t)lam * a.nleaf + sig];
        const bool bdiag = SYM && mu == nu, kdiag = SYM && lam == sig;
        const bool diag8 = EIGHT && mu == lam && nu == sig;   // keep bra pair <= ket pair
        const int64_t ma = bdiag ? nmu * (nmu + 1) / 2 : nmu * nnu;
        const int64_t mb = kdiag ? nlam * (nlam + 1) / 2 : nlam * nsig;
        // slot density blocks: g0 P[nu,lam] g1 P[mu,lam] g2 P[nu,sig] g3 P[mu,sig]
        const int rs[4] = {snu, smu, snu, smu}, cs[4] = {slam, slam, ssig, ssig};
        const int64_t total = ma * mb;
        for (int64_t q0 = 0; q0 < total; q0 += 32) {
            const int64_t q = q0 + lane;
            bool keep_any = false;
            int mask = 0;
            int64_t pa = 0, pb = 0;
            int ca = 0, cb = 0;
            if (q < total) {
                const int ia = (int)(q / mb), ib = (int)(q - (int64_t)ia * mb);
                int x, y, z, w;
                if (bdiag) tri_decode(ia, nmu, &x, &y);
                else { x = ia / nnu; y = ia - x * nnu; }
                if (kdiag) tri_decode(ib, nlam, &z, &w);
                else { z = ib / nsig; w = ib - z * nsig; }
                pa = bb + x * nnu + y;
                pb = kb + z * nsig + w;
                if (!(diag8 && ib < ia)) {
                    const double sqa = __ldg(a.sqb + pa), sqk = __ldg(a.sqk + pb);
                    const double fa = schwarz ? sqa : __ldg(a.qb + pa), fb = schwarz ? sqk : __ldg(a.qk + pb);
                    ca = a.metab[pa];
                    cb = a.metak[pb];
                    const int rowv[4] = {y, x, y, x}, colv[4] = {z, z, w, w};
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        if (!((live >> g) & 1)) continue;
                        const double pm = __ldg(a.pmax + (int64_t)(rs[g] + rowv[g]) * a.ns + cs[g] + colv[g]);
                        const double bound = __dmul_rn(__dmul_rn(fa, pm), fb);
                        if (bound >= tie_lo && bound <= tie_hi && a.tau > 0.0) {
                            ++n_tie;
                            if (TIES) tie_emit_leaf(a.ties, a.bpi, a.bpj, a.kpi, a.kpj, pa, pb, g, bound, a.tau);
                        }
                        if (bound > a.tau) {
                            keep_any = true;
                            mask |= 1 << g;
                        } else {
                            ++n_cull;
                            ledger += schwarz ? bound : __dmul_rn(__dmul_rn(sqa, pm), sqk);
                        }
                    }
                    if (SYM) {
                        // diagonal-pair weights: g1/g3 need i != j, g2/g3 need k != l
                        if (bdiag && x == y) mask &= ~0xa;
                        if (kdiag && z == w) mask &= ~0xc;
                    }
                    n_eri += keep_any;
                }
            }
            if (EMIT) {
                const unsigned bal = __ballot_sync(0xffffffffu, keep_any);
                if (bal) {
                    const uint64_t cls = (uint64_t)(((ca & 3) << 2) | (cb & 3));
                    const uint64_t selfm = (EIGHT && pa == pb) ? 1ull : 0ull;   // weight 1/2 (eightfold)
                    slab_emit(slab, a, bal, keep_any,
                              (uint64_t)pa | ((uint64_t)pb << 28) | ((uint64_t)mask << 56) | (selfm << 60),
                              (uint16_t)((cls << 8) | ((ca >> 2) << 4) | (cb >> 2)), lane);
                }
            }
        }
    }
    if (EMIT) slab_pad(slab, a, lane);
    // per-lane totals; counters are integers (order independent); the warp's
    // ledger partial has a fixed task->warp assignment and a fixed shuffle tree
    n_eri = warp_sum_ll(n_eri);
    n_cull = warp_sum_ll(n_cull);
    n_tie = warp_sum_ll(n_tie);
    ledger = warp_sum(ledger);
    if (lane == 0) {
        if (n_eri) atomic_add_ll(&a.counters[C_ERIQ], n_eri);
        if (n_cull) atomic_add_ll(&a.counters[C_CULL_LEAF], n_cull);
        if (n_tie) atomic_add_ll(&a.counters[C_TIE_LEAF], n_tie);
        if (ledger != 0.0) {
            unsigned long long limb[LEDGER_LIMBS];
            fx_from_double<LEDGER_LIMBS>(0.5 * ledger, LEDGER_SCALE, limb);
            fx_atomic_add<LEDGER_LIMBS>(a.ledger, limb);
        }
    }
}

// ---------------------------------------------------------------------------
// Hierarchical leaf screen.  Same decisions as k_screen, fewer tests:
// for a bra pair a and a ket row shell k (the "triple"), every ket pair
// b = (k, l) satisfies bound_g(a,b) = fl(fl(f_a p_g) f_b) <= fl(fl(f_a Pmax_g) Fmax_k)
// because IEEE rounding is monotone.  If that upper bound is <= tau(1 - 1e-12)
// for every live slot, the whole row is culled without per-quartet tests
// (and no quartet in it can be a tie); its culled count is exact and its
// ledger contribution is the row sum (within 1e-15 relative of the
// per-quartet sum).  Passing triples go to a per-warp queue whose entries
// are expanded lane-parallel into exact per-quartet tests.

// MS = max shells per leaf span of the system (8 for every BASELINE p-shell
// config, 10 for all-s systems at leaf size 10): smaller per-warp staging
// means more resident warps to hide the staging loads.
template <bool SYM, int MS>
struct Smem2 {
    static constexpr int NG = SYM ? 4 : 1, MP = MS * MS;
    double fa[MP], sa[MP], fb[MP], sb[MP];
    double pm[NG][MP];
    double w[SYM ? 2 : 1][SYM ? MP : 1];    // g2/g3 row ledgers: sum_{b in L_k} pm_g[r, l(b)] sb[b]
    double nvb[4 * MS], nvk[4 * MS];   // node vectors of the bra / ket leaf nodes (F entries as f),
                                       // component o of shell r at (o / NV_MAXS) * MS + r
    double z[SYM ? 2 : 1][SYM ? MP : 1];    // g2/g3: max_{b in L_k} pm_g[r, l(b)] f_b
    unsigned char ax[MP], ay[MP], acl[MP], bx[MP], by[MP], bcl[MP];
    unsigned short apl[MP], bpl[MP];
    unsigned char bstart[MS], nl[MS];
    unsigned short queue[64];
    double rmax[NG][MS];   // per slot and bra row shell: max over ket rows k of the triple factor
    double rled[NG][MS];   // per slot and bra row shell: sum over ket rows k of the triple ledger factor
    // bra pairs that pass the bra-level test: ia | (passing slots << 8) (SYM), ia (naive: slot 0 only)
    typename std::conditional<SYM, unsigned short, unsigned char>::type alist[MP];
};

template <bool SYM, int MS>
constexpr int screen2_warps() {  // static smem <= 48 KB per block
    return MS <= 8 ? (SYM ? 6 : 12) : (SYM ? 4 : 8);
}

// 1/n for the span sizes n <= 32 (fdiv's reciprocal), a constant-bank lookup
// instead of an IEEE single division per use
__constant__ float c_inv[33] = {0.f, 1.f / 1, 1.f / 2, 1.f / 3, 1.f / 4, 1.f / 5, 1.f / 6, 1.f / 7, 1.f / 8,
                                1.f / 9, 1.f / 10, 1.f / 11, 1.f / 12, 1.f / 13, 1.f / 14, 1.f / 15, 1.f / 16,
                                1.f / 17, 1.f / 18, 1.f / 19, 1.f / 20, 1.f / 21, 1.f / 22, 1.f / 23, 1.f / 24,
                                1.f / 25, 1.f / 26, 1.f / 27, 1.f / 28, 1.f / 29, 1.f / 30, 1.f / 31, 1.f / 32};

__device__ __forceinline__ int fdiv(int a, int n, float inv) {
    return __float2int_rz(((float)a + 0.5f) * inv);  // exact for a < 2^20, n <= 32
}

// EIGHT (with SYM): the eightfold driver's bra pair <= ket pair rule on bra == ket tasks
template <bool SYM, bool EMIT, int MS, bool EIGHT = false>
// (MS <= 8: 24 resident warps per SM = at most 80 registers, the measured sweet spot,
// profiles/r02_ab_eri_memory.log; the MS = 10 instances are bound by their shared memory)
__global__ void __launch_bounds__(screen2_warps<SYM, MS>() * 32, MS <= 8 ? 24 / screen2_warps<SYM, MS>() : 1) k_screen2(ScreenArgs a) {
    constexpr int NW = screen2_warps<SYM, MS>();
    __shared__ Smem2<SYM, MS> sm_all[NW];
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    Smem2<SYM, MS>& sm = sm_all[wid];
    const int64_t gw = blockIdx.x * (int64_t)NW + wid;
    const int64_t Wt = (int64_t)gridDim.x * NW;
    long long n_eri = 0, n_cull = 0, n_tie = 0;
    Slab slab{0ull, SLAB};
    double ledger = 0.0;
    const bool schwarz = a.mode == HXF_MODE_SCHWARZ;
    const double tau = a.tau;
    const double tau_skip = tau * (1.0 - 1e-12);
    // tie window |bound - tau| <= 1e-12 tau (empty for tau = 0)
    const double tie_lo = tau > 0.0 ? tau - 1e-12 * tau : 1.0, tie_hi = tau > 0.0 ? tau + 1e-12 * tau : -1.0;
#ifdef HXF_PROF_SCREEN
    long long cyc[7] = {0, 0, 0, 0, 0, 0, 0};  // staging, tables, phase 1, phase 2, cell-culled tasks, tasks, zero-survivor tasks
#define PROF_MARK(v) const long long v = clock64()
#else
#define PROF_MARK(v)
#endif
    // Runs of tblock consecutive leaf tasks per warp, so a warp's survivor slab (and after the
    // stable binning every ERI warp) holds neighbouring tasks of one bra node.  The runs are
    // dealt block-cyclically (next_run == NULL) or handed out by a device counter as warps
    // finish (the next run is requested while the current one is processed).  Either way a
    // run's ledger contribution is rounded to fixed point once per run, in a fixed shuffle
    // tree, so the ledger words do not depend on which warp took which run.
    // (32-bit run and task indices relative to t0: a chunk holds far fewer than 2^31 tasks)
    const int TB = a.tblock;
    const int ntask = (int)(a.t1 - a.t0);
    const bool dyn = a.next_run != nullptr;
    __shared__ unsigned long long s_led[NW][LEDGER_LIMBS];
    if (lane < LEDGER_LIMBS) s_led[wid][lane] = 0ull;
    __syncwarp();
    unsigned run = (unsigned)gw;
    if (dyn) {
        unsigned r0 = 0;
        if (lane == 0) r0 = atomicAdd(a.next_run, 1u);
        run = __shfl_sync(0xffffffffu, r0, 0);
    }
    while ((int64_t)run * TB < ntask) {
    unsigned pend = 0;
    if (dyn && lane == 0) pend = atomicAdd(a.next_run, 1u);
    const int tend = min(ntask, (int)(run * TB) + TB);
    for (int tl = (int)(run * TB); tl < tend; ++tl) {
        const int64_t t = a.t0 + tl;
        PROF_MARK(c_start);
        const uint64_t task = a.tasks[t];
        const int mu = task & 0x7fff, nu = (task >> 15) & 0x7fff, lam = (task >> 30) & 0x7fff,
                  sig = (task >> 45) & 0x7fff;
        int live = SYM ? (int)(task >> 60) : 1;
        const int smu = a.lslo[mu], snu = a.lslo[nu], slam = a.lslo[lam], ssig = a.lslo[sig];
        const int nmu = a.lshi[mu] - smu, nnu = a.lshi[nu] - snu, nlam = a.lshi[lam] - slam,
                  nsig = a.lshi[sig] - ssig;
        const int64_t bb = a.bra_base[(int64_t)mu * a.nleaf + nu];
        const int64_t kb = a.ket_base[(int64_t)lam * a.nleaf + sig];
        const bool bdiag = SYM && mu == nu, kdiag = SYM && lam == sig;
        const int ma = bdiag ? nmu * (nmu + 1) / 2 : nmu * nnu;
        const int mb = kdiag ? nlam * (nlam + 1) / 2 : nlam * nsig;
        // eightfold: on a bra node == ket node task only quartets with bra pair <=
        // ket pair exist (same enumeration on both sides); the bulk culls below
        // count whole blocks, so such tasks take the per-quartet path throughout
        const bool diag8 = EIGHT && mu == lam && nu == sig;
        const float inv_nnu = c_inv[nnu], inv_nsig = c_inv[nsig], inv_nlam = c_inv[nlam];
        // ---- stage density factors per live slot: g0 P[nu,lam] g1 P[mu,lam] g2 P[nu,sig] g3 P[mu,sig],
        // and the node vectors of the bra and ket leaf nodes (row / column max f, sums of s).
        // Every load of the task is issued before the first use (one memory latency per
        // task instead of one per loop trip).
        const int rs[4] = {snu, smu, snu, smu}, rn[4] = {nnu, nmu, nnu, nmu};
        const int cs[4] = {slam, slam, ssig, ssig}, cn[4] = {nlam, nlam, nsig, nsig};
        {
            constexpr int NG = Smem2<SYM, MS>::NG, NIT = (MS * MS + 31) / 32, NVI = (8 * MS + 31) / 32;
            double vp[NG][NIT], vn[NVI];
            const double* vb = bdiag ? a.nvecb_tri + (int64_t)mu * NVEC
                                     : a.nvecb + (int64_t)a.ncidb[(int64_t)mu * a.nleaf + nu] * NVEC;
            const double* vk = kdiag ? a.nveck_tri + (int64_t)lam * NVEC
                                     : a.nveck + (int64_t)a.ncidk[(int64_t)lam * a.nleaf + sig] * NVEC;
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const bool lg = (live >> g) & 1;
                const float inv = c_inv[cn[g]];
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int i = lane + 32 * u;
                    vp[g][u] = 0.0;
                    if (lg && i < rn[g] * cn[g]) {
                        const int x = fdiv(i, cn[g], inv), y = i - x * cn[g];
                        vp[g][u] = __ldg(a.pmax + (int64_t)(rs[g] + x) * a.ns + cs[g] + y);
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < NVI; ++u) {
                const int i = lane + 32 * u;
                vn[u] = 0.0;
                if (i < 8 * MS) {
                    const int h = i < 4 * MS ? i : i - 4 * MS;
                    const int o = h / MS, r = h - o * MS;
                    // F entries: max Q (literal) or its square root (Schwarz: NV_GR / NV_GC)
                    vn[u] = __ldg((i < 4 * MS ? vb : vk) + ((schwarz && o < 2) ? o + 4 : o) * NV_MAXS + r);
                }
            }
#pragma unroll
            for (int g = 0; g < NG; ++g) {
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    const int i = lane + 32 * u;
                    if (((live >> g) & 1) && i < rn[g] * cn[g]) sm.pm[g][i] = vp[g][u];
                }
            }
#pragma unroll
            for (int u = 0; u < NVI; ++u) {
                const int i = lane + 32 * u;
                if (i < 8 * MS) {
                    const int h = i < 4 * MS ? i : i - 4 * MS;
                    (i < 4 * MS ? sm.nvb : sm.nvk)[h] = vn[u];
                }
            }
        }
        __syncwarp();
        // ---- cell test: for slot g, bra row shell r and ket column shell c, every
        // quartet bound fl(fl(f_a p) f_b) <= F_A(r) p(r,c) F_B(c) (1 + 4 eps).  A task
        // with no passing cell in any live slot is culled whole (no quartet can be a
        // tie); its ledger is sum_{r,c} S_A(r) p(r,c) S_B(c) per slot.
        // A slot with no passing cell is closed for the whole task (its count and
        // ledger are added here), so the later phases stage and test the open slots only.
        if (!diag8) {
            int closed = 0;
#pragma unroll
            for (int g = 0; g < Smem2<SYM, MS>::NG; ++g) {
                if (!((live >> g) & 1)) continue;
                bool anyp = false;
                double lcell = 0.0;
                const int fo = (g == 0 || g == 2) ? MS : 0, so = fo + 2 * MS;   // F_C / F_R, S_C / S_R
                const int fk = g < 2 ? 0 : MS, sk = fk + 2 * MS;
                const float inv = c_inv[cn[g]];
#pragma unroll 1
                for (int i = lane; i < rn[g] * cn[g]; i += 32) {
                    const int r = fdiv(i, cn[g], inv), c = i - r * cn[g];
                    const double pm = sm.pm[g][i];
                    if (!(sm.nvb[fo + r] * pm * sm.nvk[fk + c] * (1.0 + 1e-14) <= tau_skip)) anyp = true;
                    lcell += sm.nvb[so + r] * pm * sm.nvk[sk + c];
                }
                if (!__any_sync(0xffffffffu, anyp)) {
                    closed |= 1 << g;
                    if (lane == 0) n_cull += (long long)ma * mb;
                    ledger += lcell;
                }
            }
            live &= ~closed;
            if (!live) {
#ifdef HXF_PROF_SCREEN
                ++cyc[4];
#endif
                __syncwarp();
                continue;
            }
        }
        // ---- stage pair factors (all loads first)
        {
            constexpr int NIT = (MS * MS + 31) / 32;
            double sqa[NIT], qa[NIT], sqk[NIT], qk[NIT];
            int mta[NIT], mtk[NIT], xa[NIT], ya[NIT], xk[NIT], yk[NIT];
#pragma unroll
            for (int u = 0; u < NIT; ++u) {
                const int i = lane + 32 * u;
                sqa[u] = qa[u] = sqk[u] = qk[u] = 0.0;
                mta[u] = mtk[u] = xa[u] = ya[u] = xk[u] = yk[u] = 0;
                if (i < ma) {
                    if (bdiag) tri_decode(i, nmu, &xa[u], &ya[u]);
                    else { xa[u] = fdiv(i, nnu, inv_nnu); ya[u] = i - xa[u] * nnu; }
                    const int64_t pid = bb + xa[u] * nnu + ya[u];
                    sqa[u] = __ldg(a.sqb + pid);
                    if (!schwarz) qa[u] = __ldg(a.qb + pid);
                    mta[u] = __ldg(a.metab + pid);
                }
                if (i < mb) {
                    if (kdiag) tri_decode(i, nlam, &xk[u], &yk[u]);
                    else { xk[u] = fdiv(i, nsig, inv_nsig); yk[u] = i - xk[u] * nsig; }
                    const int64_t pid = kb + xk[u] * nsig + yk[u];
                    sqk[u] = __ldg(a.sqk + pid);
                    if (!schwarz) qk[u] = __ldg(a.qk + pid);
                    mtk[u] = __ldg(a.metak + pid);
                }
            }
#pragma unroll
            for (int u = 0; u < NIT; ++u) {
                const int i = lane + 32 * u;
                if (i < ma) {
                    sm.sa[i] = sqa[u];
                    sm.fa[i] = schwarz ? sqa[u] : qa[u];
                    sm.ax[i] = xa[u];
                    sm.ay[i] = ya[u];
                    sm.apl[i] = xa[u] * nnu + ya[u];
                    sm.acl[i] = mta[u];
                }
                if (i < mb) {
                    sm.sb[i] = sqk[u];
                    sm.fb[i] = schwarz ? sqk[u] : qk[u];
                    sm.bx[i] = xk[u];
                    sm.by[i] = yk[u];
                    sm.bpl[i] = xk[u] * nsig + yk[u];
                    sm.bcl[i] = mtk[u];
                }
            }
        }
        // ket rows: L_k = ket pairs with row shell k (contiguous in the pair order);
        // max f and sum s over L_k are the ket node's row vectors
        if (lane < nlam) {
            const int k = lane;
            sm.bstart[k] = kdiag ? k * nlam - k * (k - 1) / 2 : k * nsig;
            sm.nl[k] = kdiag ? nlam - k : nsig;
        }
        __syncwarp();
        PROF_MARK(c_staged);
#ifdef HXF_PROF_SCREEN
        const long long n_eri_before = n_eri;
        ++cyc[5];
#endif
        if (SYM) {
            // g2/g3: row maxima over l, and row ledgers per (r, k)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int g = 2 + h;
                if (!((live >> g) & 1)) continue;
#pragma unroll 1
                for (int i = lane; i < rn[g] * nlam; i += 32) {
                    const int r = fdiv(i, nlam, inv_nlam), k = i - r * nlam;
                    const int st = kdiag ? k * nlam - k * (k - 1) / 2 : k * nsig;
                    const int n = kdiag ? nlam - k : nsig;
                    double s = 0.0, zm = 0.0;
#pragma unroll 1
                    for (int b = st; b < st + n; ++b) {
                        const double pv = sm.pm[g][r * nsig + sm.by[b]];
                        s += pv * sm.sb[b];
                        zm = fmax(zm, pv * sm.fb[b]);
                    }
                    sm.w[h][i] = s;
                    sm.z[h][i] = zm;
                }
            }
        }
        __syncwarp();
        // bra-level tables: for slot g and bra row shell r (y for g0/g2, x for g1/g3)
        //   rmax = max_k triple factor (pm_g[r,k] fbmax_k, or z),  rled = sum_k triple ledger factor
        for (int i = lane; i < Smem2<SYM, MS>::NG * MS; i += 32) {
            const int g = i / MS, r = i - g * MS;
            if (!((live >> g) & 1) || r >= rn[g]) continue;
            double m = 0.0, l = 0.0;
#pragma unroll 1
            for (int k = 0; k < nlam; ++k) {
                if (g < 2) {
                    const double pm = sm.pm[g][r * nlam + k];
                    m = fmax(m, pm * sm.nvk[k]);
                    l += pm * sm.nvk[2 * MS + k];
                } else {
                    m = fmax(m, sm.z[g - 2][r * nlam + k]);
                    l += sm.w[g - 2][r * nlam + k];
                }
            }
            sm.rmax[g][r] = m;
            sm.rled[g][r] = l;
        }
        __syncwarp();
        PROF_MARK(c_tables);
#ifdef HXF_PROF_SCREEN
        long long c_flush = 0;
#endif
        // ---- phase 0: bra pairs.  Every triple bound of bra pair a in slot g is
        // fl(fl(f_a p) f) or fl(f_a z (1 + 1e-15)) <= f_a rmax_g (1 + 4 eps), so a
        // slot with f_a rmax_g (1 + 1e-14) <= tau (1 - 1e-12) is culled for the
        // whole bra pair (every quartet bound below tau, none a tie): its count
        // and row ledger are added here and later phases test only the passing
        // slots.  A pair with no passing slot is culled whole.
        int npass = 0;
#pragma unroll 1
        for (int a0 = 0; a0 < ma; a0 += 32) {
            const int ia = a0 + lane;
            int amask = 0;
            if (ia < ma) {
                const double fa = sm.fa[ia], sa = sm.sa[ia];
                const int x = sm.ax[ia], y = sm.ay[ia];
#pragma unroll
                for (int g = 0; g < Smem2<SYM, MS>::NG; ++g) {
                    if (!((live >> g) & 1)) continue;
                    const int r = (g == 0 || g == 2) ? y : x;
                    if (diag8 || !(fa * sm.rmax[g][r] * (1.0 + 1e-14) <= tau_skip)) {
                        amask |= 1 << g;
                    } else {
                        n_cull += mb;
                        ledger += sa * sm.rled[g][r];
                    }
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, amask != 0);
            if (amask) sm.alist[npass + __popc(bal & ((1u << lane) - 1u))] = SYM ? (ia | (amask << 8)) : ia;
            npass += __popc(bal);
        }
        __syncwarp();
        // ---- phase 1: triples (a, k) of passing bra pairs; phase 2: queued triples x l, exact tests
        int qn = 0;
        const int ntrip = npass * nlam;
        const int Wl = kdiag ? nlam : nsig;       // lanes per queued triple
        const int per = 32 / Wl;                  // triples per phase-2 pass
        const int my_e = lane / Wl, my_l = lane - my_e * Wl;
        auto flush = [&](int count) {
#pragma unroll 1
            for (int e0 = 0; e0 < count; e0 += per) {
                const int e = e0 + my_e;
                bool keep_any = false;
                int mask = 0, ia = 0, ib = 0;
                if (my_e < per && e < count) {
                    const int ent = sm.queue[e];
                    ia = ent >> 8;
                    const int tmask = (ent >> 4) & 15;   // slots still open for this row
                    const int k = ent & 15;
                    if (my_l < sm.nl[k] && !(diag8 && (int)sm.bstart[k] + my_l < ia)) {
                        ib = sm.bstart[k] + my_l;
                        const double fa = sm.fa[ia], fb = sm.fb[ib];
                        const int x = sm.ax[ia], y = sm.ay[ia], z = sm.bx[ib], w = sm.by[ib];
                        const int rowv[4] = {y, x, y, x}, colv[4] = {z, z, w, w};
#pragma unroll
                        for (int g = 0; g < Smem2<SYM, MS>::NG; ++g) {
                            if (!((tmask >> g) & 1)) continue;
                            const double pm = sm.pm[g][rowv[g] * cn[g] + colv[g]];
                            const double bound = __dmul_rn(__dmul_rn(fa, pm), fb);
                            n_tie += bound >= tie_lo && bound <= tie_hi;
                            if (bound > tau) {
                                keep_any = true;
                                mask |= 1 << g;
                            } else {
                                ++n_cull;
                                ledger += schwarz ? bound : __dmul_rn(__dmul_rn(sm.sa[ia], pm), sm.sb[ib]);
                            }
                        }
                        if (SYM) {
                            const bool ij = !(bdiag && x == y), kl = !(kdiag && z == w);
                            if (!ij) mask &= ~0xa;
                            if (!kl) mask &= ~0xc;
                        }
                        n_eri += keep_any;
                    }
                }
                if (EMIT) {
                    const unsigned bal = __ballot_sync(0xffffffffu, keep_any);
                    if (bal) {
                        const uint64_t pb = (uint64_t)(bb + sm.apl[ia]);
                        const uint64_t pk = (uint64_t)(kb + sm.bpl[ib]);
                        const int ca = sm.acl[ia], cb = sm.bcl[ib];
                        const uint64_t cls = (uint64_t)(((ca & 3) << 2) | (cb & 3));
                        // bit 60: eightfold self-mirror quartet (bra pair == ket pair), weight 1/2
                        const uint64_t selfm = (EIGHT && pb == pk) ? 1ull : 0ull;
                        slab_emit(slab, a, bal, keep_any, pb | (pk << 28) | ((uint64_t)mask << 56) | (selfm << 60),
                                  (uint16_t)((cls << 8) | ((ca >> 2) << 4) | (cb >> 2)), lane);
                    }
                }
            }
        };
        // one flush call site keeps the kernel's code small (instruction cache)
        for (int t0 = 0;; t0 += 32) {
            const bool more = t0 < ntrip;
            const int tt = t0 + lane;
            int ia = 0, k = 0;
            int tmask = 0;
            if (more && tt < ntrip) {
                const int ai = fdiv(tt, nlam, inv_nlam);
                k = tt - ai * nlam;
                const int ent = sm.alist[ai];
                ia = ent & 0xff;
                const int amask = SYM ? ent >> 8 : 1;
                const double fa = sm.fa[ia], sa = sm.sa[ia], fm = sm.nvk[k];
                const int x = sm.ax[ia], y = sm.ay[ia];
#pragma unroll
                for (int g = 0; g < Smem2<SYM, MS>::NG; ++g) {
                    if (!((amask >> g) & 1)) continue;
                    double ub, led;
                    if (g < 2) {
                        const double pm = sm.pm[g][(g == 0 ? y : x) * nlam + k];
                        ub = __dmul_rn(__dmul_rn(fa, pm), fm);
                        led = __dmul_rn(sa, pm) * sm.nvk[2 * MS + k];
                    } else {
                        // fl(fl(f_a p) f_b) <= f_a max(p f_b) (1 + 4 eps): the skip
                        // threshold tau (1 - 1e-12) leaves far more slack than that
                        const int r = (g == 2) ? y : x;
                        ub = fa * sm.z[g - 2][r * nlam + k] * (1.0 + 1e-15);
                        led = sa * sm.w[g - 2][r * nlam + k];
                    }
                    if (diag8 || !(ub <= tau_skip)) {
                        tmask |= 1 << g;
                    } else {  // this slot culled for the whole row (no ties)
                        n_cull += sm.nl[k];
                        ledger += led;
                    }
                }
            }
            const bool pass = tmask != 0;
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (pass) sm.queue[qn + __popc(bal & ((1u << lane) - 1u))] = (unsigned short)((ia << 8) | (tmask << 4) | k);
            qn += __popc(bal);
            __syncwarp();
            if (qn >= 32 || (!more && qn > 0)) {
                PROF_MARK(f0);
                flush(qn);
                qn = 0;
                __syncwarp();
#ifdef HXF_PROF_SCREEN
                c_flush += clock64() - f0;
#endif
            }
            if (!more) break;
        }
        {
#ifdef HXF_PROF_SCREEN
            const long long c_end = clock64();
            cyc[0] += c_staged - c_start;
            cyc[1] += c_tables - c_staged;
            cyc[2] += c_end - c_tables - c_flush;
            cyc[3] += c_flush;
            if (__reduce_add_sync(0xffffffffu, (unsigned)(n_eri - n_eri_before)) == 0) ++cyc[6];
#endif
        }
    }
    {   // the run's ledger, rounded once, into the warp's 256-bit partial
        const double lr = warp_sum(ledger);
        ledger = 0.0;
        if (lane == 0 && lr != 0.0) {
            unsigned long long limb[LEDGER_LIMBS];
            fx_from_double<LEDGER_LIMBS>(0.5 * lr, LEDGER_SCALE, limb);
            unsigned long long carry = 0;
#pragma unroll
            for (int k = 0; k < LEDGER_LIMBS; ++k) {
                const unsigned long long x = s_led[wid][k], y = x + limb[k], z = y + carry;
                carry = (unsigned long long)(y < x) + (unsigned long long)(z < y);
                s_led[wid][k] = z;
            }
        }
    }
    run = dyn ? __shfl_sync(0xffffffffu, pend, 0) : run + (unsigned)Wt;
    }
    if (EMIT) slab_pad(slab, a, lane);
    n_eri = warp_sum_ll(n_eri);
    n_cull = warp_sum_ll(n_cull);
    n_tie = warp_sum_ll(n_tie);
    if (lane == 0) {
#ifdef HXF_PROF_SCREEN
        for (int k = 0; k < 4; ++k) atomic_add_ll(&a.counters[C_DBG0 + k], cyc[k]);
        for (int k = 4; k < 7; ++k) atomic_add_ll(&a.counters[C_DBG0 + k], cyc[k]);
#endif
        if (n_eri) atomic_add_ll(&a.counters[C_ERIQ], n_eri);
        if (n_cull) atomic_add_ll(&a.counters[C_CULL_LEAF], n_cull);
        if (n_tie) atomic_add_ll(&a.counters[C_TIE_LEAF], n_tie);
        unsigned long long limb[LEDGER_LIMBS];
        bool any = false;
#pragma unroll
        for (int k = 0; k < LEDGER_LIMBS; ++k) {
            limb[k] = s_led[wid][k];
            any |= limb[k] != 0ull;
        }
        if (any) fx_atomic_add<LEDGER_LIMBS>(a.ledger, limb);
    }
}

// Leaf-screen algorithmic bytes: per leaf task 8 (m_bra + m_ket) B of Q
// plus 8 n_row n_col B of the |P| block per live slot.  A measurement pass over the leaf
// task list (hxf_exchange_opts.count_screen_bytes), not part of a normal build.
__global__ void k_screen_bytes(const uint64_t* tasks, int64_t n, const int* lslo, const int* lshi, int sym,
                               long long* counters) {
    long long b = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t task = tasks[t];
        const int mu = task & 0x7fff, nu = (task >> 15) & 0x7fff, lam = (task >> 30) & 0x7fff,
                  sig = (task >> 45) & 0x7fff;
        const int live = sym ? (int)(task >> 60) : 1;
        const int nmu = lshi[mu] - lslo[mu], nnu = lshi[nu] - lslo[nu], nlam = lshi[lam] - lslo[lam],
                  nsig = lshi[sig] - lslo[sig];
        const long long ma = (sym && mu == nu) ? nmu * (nmu + 1) / 2 : nmu * nnu;
        const long long mb = (sym && lam == sig) ? nlam * (nlam + 1) / 2 : nlam * nsig;
        b += 8 * (ma + mb) + 8 * (((live & 1) ? nnu * nlam : 0) + ((live & 2) ? nmu * nlam : 0) +
                                  ((live & 4) ? nnu * nsig : 0) + ((live & 8) ? nmu * nsig : 0));
    }
    b = warp_sum_ll(b);
    if ((threadIdx.x & 31) == 0 && b) atomic_add_ll(&counters[C_SCREEN_BYTES], b);
}

struct EriArgs {
    const uint64_t* rec;
    int64_t n;
    const int* bpi;
    const int* bpj;
    const int64_t* bppoff;
    const PrimPair* bpp;
    const int* kpi;
    const int* kpj;
    const int64_t* kppoff;
    const PrimPair* kpp;
    const int4* binfo;
    const int4* kinfo;
    const int4* bfinfo;   // far-field kernels: collapsed same-centre (ss| pairs (k_prune_pairs)
    const int4* kfinfo;
    const double3* ctr;
    const int* fn;
    const double* P;
    int nfn;
    int S;
    unsigned long long* K;
    long long* counters;
    const int64_t* dbounds;  // non-NULL: this class's record range is read on the device
    int64_t n_bpairs, n_kpairs, n_bprim, n_kprim;   // table sizes (HXF_DEBUG_BOUNDS checks)
};

__device__ __forceinline__ void k_add(const EriArgs& e, int row, int col, double v) {
    if (v == 0.0) return;
#ifdef HXF_EXP_NOATOM  // timing experiment: no K traffic (results wrong)
    if (v == 1.2345) e.K[0] = 1;
    return;
#endif
    if (!HXF_BCHECK(row >= 0 && row < e.nfn && col >= 0 && col < e.nfn, e.counters)) return;
    k_fixed_add(e.K + ((int64_t)row * e.nfn + col), v, e.S);
}

// Warp-combined K flush (HXF_KCOMBINE, north star item 4): the lanes of a warp whose
// contribution goes to the same K element (the records of one (bra pair, ket row)
// run share K[mu,lam] and K[nu,lam]) are summed first -- in fixed point, each value
// already rounded as the direct path rounds it, so K stays bitwise the same -- and
// one lane issues a single reduction per distinct element.  Called by all 32 lanes.
__device__ __forceinline__ void k_add_warp(const EriArgs& e, bool on, int row, int col, double v) {
    const int lane = threadIdx.x & 31;
    long long fv = 0, key = -1 - lane;
    if (on) {
        fv = __double2ll_rn(ldexp(v, e.S));
        key = (long long)row * e.nfn + col;
    }
    const unsigned peers = __match_any_sync(0xffffffffu, key);
    const bool leader = (__ffs(peers) - 1) == lane;
    int rel = __popc(peers & ((1u << lane) - 1u));   // my position among my peers
    unsigned rest = peers & (0xfffffffeu << lane);    // the peers above me
    while (__any_sync(0xffffffffu, rest != 0)) {      // log2(largest group) steps
        const int next = __ffs(rest);
        const long long t = __shfl_sync(0xffffffffu, fv, next ? next - 1 : lane);
        if (next) fv += t;
        const bool done = rel & 1;
        rest &= __ballot_sync(0xffffffffu, !done);
        rel >>= 1;
    }
    if (leader && on && fv) atomicAdd(e.K + key, (unsigned long long)fv);
}

// (re-tuned after the bra-node-major leaf order, profiles/r02_ab_locality.log: with the memory
// path relieved the near (ss|ss) kernel prefers 2 blocks / 255 registers, the far-field kernels
// more resident blocks: c5 ERI kernels 3366 -> 3188 ms)
#ifndef HXF_ERI_MINB0
#define HXF_ERI_MINB0 2
#endif

#ifndef HXF_ERI_MINB1
#define HXF_ERI_MINB1 2
#endif
// classes whose bit (LA<<3 | LB<<2 | LC<<1 | LD) is set in HXF_ERI_MINB3_MASK are
// compiled for 3 resident blocks per SM (<= 168 registers) instead of HXF_ERI_MINB1
#ifndef HXF_ERI_MINB3_MASK
#define HXF_ERI_MINB3_MASK 0
#endif
__host__ __device__ constexpr int eri_min_blocks(int la, int lb, int lc, int ld) {
    return (la + lb + lc + ld) == 0 ? HXF_ERI_MINB0
           : ((HXF_ERI_MINB3_MASK >> ((la << 3) | (lb << 2) | (lc << 1) | ld)) & 1) ? 3
                                                                                   : HXF_ERI_MINB1;
}
// far-field kernels: no Boys table and shorter dependency chains, so more
// resident blocks ((ss|ss): 6 = <= 80 registers; p classes 3; measured 4/5/6/8 and 2/3/4)
#ifndef HXF_ERI_FAR_MINB0
#define HXF_ERI_FAR_MINB0 6
#endif
#ifndef HXF_ERI_FAR_MINB1
#define HXF_ERI_FAR_MINB1 3
#endif
__host__ __device__ constexpr int eri_far_min_blocks(int la, int lb, int lc, int ld) {
    return (la + lb + lc + ld) == 0 ? HXF_ERI_FAR_MINB0 : HXF_ERI_FAR_MINB1;
}
template <int LA, int LB, int LC, int LD, bool FAR>
__global__ void __launch_bounds__(128, FAR ? eri_far_min_blocks(LA, LB, LC, LD) : eri_min_blocks(LA, LB, LC, LD))
    k_eri(EriArgs e) {
    typedef Eri<LA, LB, LC, LD> E;
    constexpr int NI = E::NI, NJ = E::NJ, NK = E::NK, NL = E::NL;
    constexpr int CLS = (LA << 3) | (LB << 2) | (LC << 1) | LD;
    constexpr int K0 = KEY_OF(FAR, CLS);
    if (e.dbounds) {  // asynchronous launch: range from the sorted keys' bounds
        const int64_t b0 = e.dbounds[K0];
        e.n = e.dbounds[K0 + KEY_CLASS_SPAN] - b0;
        e.rec += b0;
        if (e.n <= 0) return;
    }
    extern __shared__ __align__(16) double s_tab[];
    if (!FAR) boys_eri_table_to_smem<E::L>(s_tab);
    long long nprim = 0, nq = 0;
#ifdef HXF_KCOMBINE
    // warp-uniform trip count: every lane reaches the combined flush
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t - (threadIdx.x & 31) < e.n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = t < e.n ? e.rec[t] : 0ull;
        const int mask = (int)((r >> 56) & 0xf);
        int fi = 0, fj = 0, fk = 0, fl = 0;
        double out[NI * NJ * NK * NL];
        double half = -0.5;
        if (mask) {
            const int64_t pb = (int64_t)(r & 0xfffffff), pk = (int64_t)((r >> 28) & 0xfffffff);
            const int4 ib = __ldg((FAR ? e.bfinfo : e.binfo) + pb), ik = __ldg((FAR ? e.kfinfo : e.kinfo) + pk);
            const int nb = ib.w, nk = ik.w;
            nprim += (long long)nb * nk;
            nq += 1;
            double3 A{0, 0, 0}, B{0, 0, 0}, C{0, 0, 0}, D{0, 0, 0};
            if (LA | LB) { A = e.ctr[e.bpi[pb]]; B = e.ctr[e.bpj[pb]]; }
            if (LC | LD) { C = e.ctr[e.kpi[pk]]; D = e.ctr[e.kpj[pk]]; }
            E::template eval<FAR>(e.bpp + ib.z, nb, e.kpp + ik.z, nk, A, B, C, D, s_tab, out);
            fi = ib.x; fj = ib.y; fk = ik.x; fl = ik.y;
            if constexpr (LA == LC && LB == LD) half = ((r >> 60) & 1) ? -0.25 : -0.5;
        }
        const int64_t n = e.nfn;
        const double* P = e.P;
#define OUT(x, y, z, w) out[(((x) * NJ + (y)) * NK + (z)) * NL + (w)]
        if (__any_sync(0xffffffffu, mask & 1)) {  // K[mu,sig] <- P[nu,lam]
            const bool on = mask & 1;
            for (int x = 0; x < NI; ++x)
                for (int w = 0; w < NL; ++w) {
                    double s = 0.0;
                    if (on)
                        for (int y = 0; y < NJ; ++y)
                            for (int z = 0; z < NK; ++z) s += __ldg(P + (fj + y) * n + fk + z) * OUT(x, y, z, w);
                    k_add_warp(e, on, fi + x, fl + w, half * s);
                }
        }
        if (__any_sync(0xffffffffu, mask & 2)) {  // K[nu,sig] <- P[mu,lam]
            const bool on = mask & 2;
            for (int y = 0; y < NJ; ++y)
                for (int w = 0; w < NL; ++w) {
                    double s = 0.0;
                    if (on)
                        for (int x = 0; x < NI; ++x)
                            for (int z = 0; z < NK; ++z) s += __ldg(P + (fi + x) * n + fk + z) * OUT(x, y, z, w);
                    k_add_warp(e, on, fj + y, fl + w, half * s);
                }
        }
        if (__any_sync(0xffffffffu, mask & 4)) {  // K[mu,lam] <- P[nu,sig]
            const bool on = mask & 4;
            for (int x = 0; x < NI; ++x)
                for (int z = 0; z < NK; ++z) {
                    double s = 0.0;
                    if (on)
                        for (int y = 0; y < NJ; ++y)
                            for (int w = 0; w < NL; ++w) s += __ldg(P + (fj + y) * n + fl + w) * OUT(x, y, z, w);
                    k_add_warp(e, on, fi + x, fk + z, half * s);
                }
        }
        if (__any_sync(0xffffffffu, mask & 8)) {  // K[nu,lam] <- P[mu,sig]
            const bool on = mask & 8;
            for (int y = 0; y < NJ; ++y)
                for (int z = 0; z < NK; ++z) {
                    double s = 0.0;
                    if (on)
                        for (int x = 0; x < NI; ++x)
                            for (int w = 0; w < NL; ++w) s += __ldg(P + (fi + x) * n + fl + w) * OUT(x, y, z, w);
                    k_add_warp(e, on, fj + y, fk + z, half * s);
                }
        }
#undef OUT
    }
#else
    // (Measured and not kept, profiles/r02_ab_eri_memory.log: a software pipeline over the
    // thread's records, L1 prefetch of the bra primitives, bra primitives two iterations
    // ahead, more resident far-field blocks -- all +0.4 .. +3.4 % on the ERI stage.)
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < e.n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = e.rec[t];
        const int mask = (int)((r >> 56) & 0xf);
        if (mask) {
            const int64_t pb = (int64_t)(r & 0xfffffff), pk = (int64_t)((r >> 28) & 0xfffffff);
            if (!HXF_BCHECK(pb < e.n_bpairs && pk < e.n_kpairs, e.counters)) continue;
            // one 16-byte record per pair: function offsets, primitive-pair range
            const int4 ib = __ldg((FAR ? e.bfinfo : e.binfo) + pb), ik = __ldg((FAR ? e.kfinfo : e.kinfo) + pk);
            const int nb = ib.w, nk = ik.w;
            if (!HXF_BCHECK(nb >= 1 && nk >= 1 && ib.z >= 0 && ik.z >= 0 && (int64_t)ib.z + nb <= e.n_bprim &&
                                (int64_t)ik.z + nk <= e.n_kprim,
                            e.counters))
                continue;
            nprim += (long long)nb * nk;
            nq += 1;
            double out[NI * NJ * NK * NL];
            double3 A{0, 0, 0}, B{0, 0, 0}, C{0, 0, 0}, D{0, 0, 0};
            if (LA | LB) { A = e.ctr[e.bpi[pb]]; B = e.ctr[e.bpj[pb]]; }
            if (LC | LD) { C = e.ctr[e.kpi[pk]]; D = e.ctr[e.kpj[pk]]; }
            const int fi = ib.x, fj = ib.y, fk = ik.x, fl = ik.y;
            const int64_t n = e.nfn;
            const double* P = e.P;
            // (ss|ss): the four density elements are requested before the primitive loops
            double pv[4] = {0.0, 0.0, 0.0, 0.0};
            if constexpr (NI * NJ * NK * NL == 1) {
                if (mask & 1) pv[0] = __ldg(P + fj * n + fk);
                if (mask & 2) pv[1] = __ldg(P + fi * n + fk);
                if (mask & 4) pv[2] = __ldg(P + fj * n + fl);
                if (mask & 8) pv[3] = __ldg(P + fi * n + fl);
            }
#ifdef HXF_EXP_NOPRIM  // timing experiment: skip the primitive loops (results wrong)
            for (int q = 0; q < NI * NJ * NK * NL; ++q) out[q] = e.bpp[ib.z].c * e.kpp[ik.z].c;
#else
            E::template eval<FAR>(e.bpp + ib.z, nb, e.kpp + ik.z, nk, A, B, C, D, s_tab, out);
#endif
            // -1/2 exchange factor; eightfold: the self-mirror quartet (bra pair ==
            // ket pair, record bit 60, only in classes with bra class == ket class)
            // enters A once and K = A + A^T, so it carries 1/2
            double half = -0.5;
            if constexpr (LA == LC && LB == LD) half = ((r >> 60) & 1) ? -0.25 : -0.5;
            if constexpr (NI * NJ * NK * NL == 1) {
                const double v = half * out[0];
                if (mask & 1) k_add(e, fi, fl, pv[0] * v);
                if (mask & 2) k_add(e, fj, fl, pv[1] * v);
                if (mask & 4) k_add(e, fi, fk, pv[2] * v);
                if (mask & 8) k_add(e, fj, fk, pv[3] * v);
            } else {
#define OUT(x, y, z, w) out[(((x) * NJ + (y)) * NK + (z)) * NL + (w)]
            if (mask & 1) {  // K[mu,sig] <- P[nu,lam]
                for (int x = 0; x < NI; ++x)
                    for (int w = 0; w < NL; ++w) {
                        double s = 0.0;
                        for (int y = 0; y < NJ; ++y)
                            for (int z = 0; z < NK; ++z) s += __ldg(P + (fj + y) * n + fk + z) * OUT(x, y, z, w);
                        k_add(e, fi + x, fl + w, half * s);
                    }
            }
            if (mask & 2) {  // K[nu,sig] <- P[mu,lam]
                for (int y = 0; y < NJ; ++y)
                    for (int w = 0; w < NL; ++w) {
                        double s = 0.0;
                        for (int x = 0; x < NI; ++x)
                            for (int z = 0; z < NK; ++z) s += __ldg(P + (fi + x) * n + fk + z) * OUT(x, y, z, w);
                        k_add(e, fj + y, fl + w, half * s);
                    }
            }
            if (mask & 4) {  // K[mu,lam] <- P[nu,sig]
                for (int x = 0; x < NI; ++x)
                    for (int z = 0; z < NK; ++z) {
                        double s = 0.0;
                        for (int y = 0; y < NJ; ++y)
                            for (int w = 0; w < NL; ++w) s += __ldg(P + (fj + y) * n + fl + w) * OUT(x, y, z, w);
                        k_add(e, fi + x, fk + z, half * s);
                    }
            }
            if (mask & 8) {  // K[nu,lam] <- P[mu,sig]
                for (int y = 0; y < NJ; ++y)
                    for (int z = 0; z < NK; ++z) {
                        double s = 0.0;
                        for (int x = 0; x < NI; ++x)
                            for (int w = 0; w < NL; ++w) s += __ldg(P + (fi + x) * n + fl + w) * OUT(x, y, z, w);
                        k_add(e, fj + y, fk + z, half * s);
                    }
            }
#undef OUT
            }
        }
    }
#endif
    nq = warp_sum_ll(nq);
    nprim = warp_sum_ll(nprim);
    if ((threadIdx.x & 31) == 0 && nprim) {
        atomic_add_ll(&e.counters[C_PRIMQ], nprim);
        atomic_add_ll(&e.counters[C_CLSPQ0 + CLS], nprim);
        atomic_add_ll(&e.counters[C_CLSQ0 + CLS], nq);
        if (FAR) {
            atomic_add_ll(&e.counters[C_DBG0 + 0], nq);
            atomic_add_ll(&e.counters[C_DBG0 + 1], nprim);
        }
    }
}

// Survivor binning: a stable counting sort by ERI bin in four kernels (no library sort).
//
// A column is the contiguous record run of one block of BINB_WARPS warps, walked in tiles of
// BINB_WARPS x 32 x BINB_ITEMS records; warp w owns records [w, w + 1) x 32 x BINB_ITEMS of a
// tile.
//
// k_binb_classify per-quartet far-field test + final bin id, written over the screen's key,
//                 and the column's histogram (shared-memory atomics: counting needs no order).
//                 The far-field decision is a function of the quartet alone (the two pairs'
//                 enclosing spheres, k_pair_geo), so every driver (naive, fourfold, eightfold,
//                 the direct twin) evaluates a given quartet with the same arithmetic.
// k_bin_rowscan   per bin: exclusive scan over the columns, in place, and the bin total.
// k_bin_scan      bin starts from the totals: the ERI kernels' record ranges.
// k_binb_scatter  all warps of a block load their records of the tile at once, then take turns
//                 (warp order, a block barrier per turn) to reserve slots from the block's
//                 shared running counters: slot = bin start + column offset + running count +
//                 rank among the lanes of the same bin (__match_any_sync).  The order inside a
//                 bin is exactly the screen's order (stable), which is the locality the ERI
//                 kernels live on (neighbouring records = neighbouring leaf tasks of one bra
//                 node).
// Traffic: 10 B read + 2 B written, then 10 B read + 8 B written per record.
// History (profiles/r02_ab_locality.log): CUB radix sort 448 ms per c5 build; warp columns
// with private counters 489-504 ms (20 warps per SM bound the loads in flight, 1.5 M slow
// (column, bin) write cursors lose partial sectors from L2); block columns 334 ms.
struct BinGeo {
    const float4* bgeo;
    const float* bgip;
    const float4* kgeo;
    const float* kgip;
    const uint8_t* bfcnt;
    const uint8_t* kfcnt;
    int do_far;
};

__device__ __forceinline__ int eri_bin_of(uint16_t key, uint64_t r, const BinGeo& g) {
    if (key == SENTINEL_KEY) return ERI_NBINS;
    const int64_t pb = (int64_t)(r & 0xfffffff), pk = (int64_t)((r >> 28) & 0xfffffff);
    const int cls = (key >> 8) & 15;   // the screen's key: class << 8 | nb-1 << 4 | nk-1
    int nb1 = (key >> 4) & 15, nk1 = key & 15, far = 0;
    if (g.do_far) {
        const int L = __popc(cls);
        const float4 gb = __ldg(g.bgeo + pb), gk = __ldg(g.kgeo + pk);
        const float ip = __ldg(g.bgip + pb) + __ldg(g.kgip + pk);
        const float dx = gb.x - gk.x, dy = gb.y - gk.y, dz = gb.z - gk.z;
        const float d = sqrtf(dx * dx + dy * dy + dz * dz) * (1.0f - 1e-5f) - gb.w - gk.w;
        // a far quartet sorts by its far-field primitive counts (1 for a collapsed pair)
        if (d > 0.0f && d * d >= (float)(boys_far_t(L) * 1.0001) * ip) {
            far = 1;
            nb1 = __ldg(g.bfcnt + pb);
            nk1 = __ldg(g.kfcnt + pk);
        }
    }
    return ((far * 16 + cls) * 9 + nb1) * 9 + nk1;
}

// per bin (one warp each): exclusive scan of the row of column counts, in place; the row total
__global__ void __launch_bounds__(256) k_bin_rowscan(unsigned* __restrict__ hist, int ncol, long long* __restrict__ total) {
    const int b = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (b > ERI_NBINS) return;
    unsigned* row = hist + (int64_t)b * ncol;
    unsigned run = 0;
    for (int k0 = 0; k0 < ncol; k0 += 32) {
        const int k = k0 + lane;
        const unsigned v = k < ncol ? row[k] : 0u;
        unsigned inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned u = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += u;
        }
        if (k < ncol) row[k] = run + inc - v;
        run += __shfl_sync(0xffffffffu, inc, 31);
    }
    if (lane == 0) total[b] = run;
}

// bin starts from the bin totals (one block; ERI_NBINS + 1 totals, the scan is serial in
// shared memory: ~10 us)
__global__ void __launch_bounds__(1024) k_bin_scan(const long long* __restrict__ total, int64_t* __restrict__ bounds) {
    __shared__ long long tot[ERI_NBINS + 2];
    for (int b = threadIdx.x; b <= ERI_NBINS; b += 1024) tot[b] = total[b];
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int b = 0; b <= ERI_NBINS; ++b) {
            const long long c = tot[b];
            tot[b] = run;
            run += c;
        }
        tot[ERI_NBINS + 1] = run;
    }
    __syncthreads();
    for (int b = threadIdx.x; b <= ERI_NBINS + 1; b += 1024) bounds[b] = tot[b];
}

#define BINB_WARPS 8
// 4 records per thread per tile and 40 registers (6 resident blocks) measured best:
// 8 / 68 registers 403 ms, 8 / 64 370, 4 / 40 334, 4 / 32 349, 2 / 32 343
#ifndef BINB_ITEMS
#define BINB_ITEMS 4
#endif
#ifndef BINB_MINB
#define BINB_MINB 6
#endif
#define BINB_TILE (BINB_WARPS * 32 * BINB_ITEMS)

__global__ void __launch_bounds__(BINB_WARPS * 32, BINB_MINB) k_binb_classify(
    const uint64_t* __restrict__ rec, uint16_t* __restrict__ keys, int64_t n, int64_t seg, BinGeo g,
    unsigned* __restrict__ hist) {
    __shared__ unsigned h[ERI_NBINS + 1];
    for (int i = threadIdx.x; i <= ERI_NBINS; i += blockDim.x) h[i] = 0;
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = blockIdx.x * seg, hi = min(n, lo + seg);
    for (int64_t tile = lo; tile < hi; tile += BINB_TILE) {
        const int64_t w0 = tile + (int64_t)wid * 32 * BINB_ITEMS;
        uint16_t key[BINB_ITEMS];
        uint64_t r[BINB_ITEMS];
#pragma unroll
        for (int u = 0; u < BINB_ITEMS; ++u) {
            const int64_t t = w0 + 32 * u + lane;
            key[u] = t < hi ? keys[t] : SENTINEL_KEY;
            r[u] = t < hi ? rec[t] : 0ull;
        }
        int bin[BINB_ITEMS];
#pragma unroll
        for (int u = 0; u < BINB_ITEMS; ++u) bin[u] = eri_bin_of(key[u], r[u], g);
#pragma unroll
        for (int u = 0; u < BINB_ITEMS; ++u) {
            const int64_t t = w0 + 32 * u + lane;
            const bool on = t < hi;
            if (on) keys[t] = (uint16_t)bin[u];
            const int b = on ? bin[u] : -1 - lane;   // out of range: a group of its own, not counted
            const unsigned peers = __match_any_sync(0xffffffffu, b);
            if (on && (__ffs(peers) - 1) == lane) atomicAdd(&h[b], (unsigned)__popc(peers));   // counting: any order
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i <= ERI_NBINS; i += blockDim.x) hist[(int64_t)i * gridDim.x + blockIdx.x] = h[i];
}

__global__ void __launch_bounds__(BINB_WARPS * 32, BINB_MINB) k_binb_scatter(
    const uint64_t* __restrict__ rec, const uint16_t* __restrict__ keys, int64_t n, int64_t seg,
    const unsigned* __restrict__ hist, const int64_t* __restrict__ bounds, uint64_t* __restrict__ out) {
    // next free slot of this column's run in each bin, relative to the bin start (< 2^29 per chunk)
    __shared__ unsigned pos[ERI_NBINS + 1];
    for (int i = threadIdx.x; i <= ERI_NBINS; i += blockDim.x) pos[i] = hist[(int64_t)i * gridDim.x + blockIdx.x];
    __syncthreads();
    const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t lo = blockIdx.x * seg, hi = min(n, lo + seg);
    for (int64_t tile = lo; tile < hi; tile += BINB_TILE) {   // block-uniform trip count
        const int64_t w0 = tile + (int64_t)wid * 32 * BINB_ITEMS;
        int bin[BINB_ITEMS];
        uint64_t r[BINB_ITEMS];
#pragma unroll
        for (int u = 0; u < BINB_ITEMS; ++u) {
            const int64_t t = w0 + 32 * u + lane;
            bin[u] = t < hi ? (int)keys[t] : -1 - lane;
            r[u] = t < hi ? rec[t] : 0ull;
        }
        unsigned dst[BINB_ITEMS];
        for (int turn = 0; turn < BINB_WARPS; ++turn) {
            if (turn == wid) {
#pragma unroll
                for (int u = 0; u < BINB_ITEMS; ++u) {
                    const int b = bin[u];
                    const unsigned peers = __match_any_sync(0xffffffffu, b);
                    const int leader = __ffs(peers) - 1;
                    unsigned base = 0;
                    if (b >= 0 && leader == lane) {
                        base = pos[b];
                        pos[b] = base + (unsigned)__popc(peers);
                    }
                    __syncwarp();
                    base = __shfl_sync(0xffffffffu, base, leader);
                    dst[u] = base + __popc(peers & ((1u << lane) - 1u));
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int u = 0; u < BINB_ITEMS; ++u)
            if (bin[u] >= 0) out[bounds[bin[u]] + dst[u]] = r[u];
    }
}

__global__ void k_log(const uint64_t* rec, int64_t n, const int* bpi, const int* bpj, const int* kpi,
                      const int* kpj, int32_t* log, int64_t cap, unsigned long long* fill) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t r = rec[t];
    if (r == SENTINEL_REC) return;  // slab padding
    const int64_t pb = (int64_t)(r & 0xfffffff), pk = (int64_t)((r >> 28) & 0xfffffff);
    const unsigned long long pos = atomicAdd(fill, 1ull);
    if ((int64_t)pos < cap) {
        log[4 * pos + 0] = bpi[pb];
        log[4 * pos + 1] = bpj[pb];
        log[4 * pos + 2] = kpi[pk];
        log[4 * pos + 3] = kpj[pk];
    }
}

// SplitMix64 finaliser (basis.py:112-136 mixes the same way)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// order-independent digest of the evaluated tuples (the k_log tuples);
// eightfold: each quartet oriented with (i,j) <= (k,l) (oracle/direct_digest.c)
__global__ void k_digest(const uint64_t* rec, int64_t n, const int* bpi, const int* bpj, const int* kpi,
                         const int* kpj, uint64_t ns, int mod, int rem, int eight, unsigned long long* dg) {
    unsigned long long c = 0, h1 = 0, h2 = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n;
         t += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t r = rec[t];
        if (r == SENTINEL_REC) continue;
        const int64_t pb = (int64_t)(r & 0xfffffff), pk = (int64_t)((r >> 28) & 0xfffffff);
        uint64_t i = bpi[pb], j = bpj[pb], k = kpi[pk], l = kpj[pk];
        if (eight && (i > k || (i == k && j > l))) {
            uint64_t x = i; i = k; k = x;
            x = j; j = l; l = x;
        }
        if (mod > 1 && (int)(i % (uint64_t)mod) != rem) continue;
        const uint64_t h = mix64(((i * ns + j) * ns + k) * ns + l);
        c += 1;
        h1 += h;
        h2 += mix64(h);
    }
    c = (unsigned long long)warp_sum_ll((long long)c);
    h1 = (unsigned long long)warp_sum_ll((long long)h1);
    h2 = (unsigned long long)warp_sum_ll((long long)h2);
    if ((threadIdx.x & 31) == 0 && c) {
        atomicAdd(dg + 0, c);
        atomicAdd(dg + 1, h1);
        atomicAdd(dg + 2, h2);
    }
}

__global__ void k_fx_to_double(const unsigned long long* Kfx, int64_t n2, int S, double* K) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n2;
         t += (int64_t)gridDim.x * blockDim.x)
        K[t] = k_fixed_value(Kfx + t, S);
}

// eightfold epilogue: A + A^T on the fixed-point accumulator (integer, exact)
__global__ void k_fold_fx(unsigned long long* K, int n) {
    const int64_t n2 = (int64_t)n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n2;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / n), j = (int)(t % n);
        if (i < j) {
            const int64_t u = (int64_t)j * n + i;
            const unsigned long long v = K[t] + K[u];
            K[t] = v;
            K[u] = v;
        } else if (i == j) {
            K[t] = K[t] * 2ull;
        }
    }
}

__global__ void k_asym(const double* K, int n, unsigned long long* out) {
    double m = 0.0;
    const int64_t n2 = (int64_t)n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n2;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / n), j = (int)(t % n);
        if (i < j) m = fmax(m, fabs(K[t] - K[(int64_t)j * n + i]));
    }
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void k_symmetrize(double* K, int n) {
    const int64_t n2 = (int64_t)n * n;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < n2;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(t / n), j = (int)(t % n);
        if (i < j) {
            const int64_t u = (int64_t)j * n + i;
            const double v = 0.5 * (K[t] + K[u]);
            K[t] = v;
            K[u] = v;
        }
    }
}

template <typename T>
T* lalloc(size_t n, cudaStream_t st) {
    if (n == 0) n = 1;
    return (T*)hxf_cache_alloc(n * sizeof(T), st);
}

// persistent grid: every block stages its Boys table once, then strides
template <int A, int B, int C, int D, bool FAR>
void launch_eri(const EriArgs& e, cudaStream_t st) {
    // the far-field kernels need no Boys table
    constexpr int TB = FAR ? 0 : boys_eri_tab_bytes(A + B + C + D);
    static int per_sm = -1, sms = 0;
    if (per_sm < 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_eri<A, B, C, D, FAR>, cudaFuncAttributeMaxDynamicSharedMemorySize, TB);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_eri<A, B, C, D, FAR>, 128, TB);
        if (const char* cap = getenv("HXF_ERI_PERSM")) per_sm = std::min(per_sm, atoi(cap));
        per_sm = std::max(per_sm, 1);
    }
    const int64_t want = e.dbounds ? (int64_t)sms * per_sm : (e.n + 127) / 128;
    const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));
    k_eri<A, B, C, D, FAR><<<g, 128, TB, st>>>(e);
    note_launch();
}

void launch_eri_class(int cls, bool far, const EriArgs& e, cudaStream_t st) {
    if (!e.n && !e.dbounds) return;
    switch (cls) {
#define C(a, b, c, d) \
    case (a << 3) | (b << 2) | (c << 1) | d: \
        if (far) launch_eri<a, b, c, d, true>(e, st); else launch_eri<a, b, c, d, false>(e, st); break;
        C(0, 0, 0, 0) C(0, 0, 0, 1) C(0, 0, 1, 0) C(0, 0, 1, 1)
        C(0, 1, 0, 0) C(0, 1, 0, 1) C(0, 1, 1, 0) C(0, 1, 1, 1)
        C(1, 0, 0, 0) C(1, 0, 0, 1) C(1, 0, 1, 0) C(1, 0, 1, 1)
        C(1, 1, 0, 0) C(1, 1, 0, 1) C(1, 1, 1, 0) C(1, 1, 1, 1)
#undef C
    }
}

thread_local double g_timings[8];

struct SurvivorBufs {
    uint64_t *rec, *rec2;   // screen order; binned
    uint16_t* keys;
    unsigned* hist;         // (ERI_NBINS + 1) x bin_blocks (columns) counts, then first slots
    int bin_blocks;
    int64_t* dbounds;       // ERI_NBINS + 2 bin starts (slab padding last)
    // per-pair spheres for the per-quartet far-field pass (NULL: skip it)
    const float4* bgeo = nullptr;
    const float4* kgeo = nullptr;
    const float* bgip = nullptr;
    const float* kgip = nullptr;
    const uint8_t* bfcnt = nullptr;   // far-field primitive count - 1 per pair (EriTables::fcnt)
    const uint8_t* kfcnt = nullptr;
};

struct Timer {
    cudaEvent_t a, b;
    cudaStream_t st;
    explicit Timer(cudaStream_t s) : st(s) {
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, st);
    }
    float stop() {
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        return ms;
    }
};

// helper streams of the ERI stage (per host thread and device; created on first use)
struct EriStreams {
    cudaStream_t s[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t fork = nullptr, join[3] = {nullptr, nullptr, nullptr};
    int dev = -1;
    void ensure() {
        int d = 0;
        cudaGetDevice(&d);
        if (dev == d) return;
        for (int k = 0; k < 3; ++k) {
            cudaStreamCreateWithFlags(&s[k], cudaStreamNonBlocking);
            cudaEventCreateWithFlags(&join[k], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        dev = d;
    }
};
EriStreams& eri_streams() {
    thread_local EriStreams x;
    return x;
}

// bin one chunk of survivors by (far, class, nb, nk) and run the per-class ERI
// kernels over the binned copy, without a host synchronisation: every class
// kernel reads its record range from the device-side bin starts (empty classes
// exit at once)
void eri_sorted_stage_async(EriArgs e, const SurvivorBufs& b, int64_t nrec, cudaStream_t st,
                            cudaEvent_t after_sort = nullptr) {
    long long* total = reinterpret_cast<long long*>(b.dbounds + ERI_NBINS + 2);
    const BinGeo geo{b.bgeo, b.bgip, b.kgeo, b.kgip, b.bfcnt, b.kfcnt, (b.bgeo && !HXF_ERI_NOFAR) ? 1 : 0};
    // one column per block; small chunks (c1 / c2: a few tiles) take only the blocks they fill
    const int G = (int)std::max<int64_t>(1, std::min<int64_t>(b.bin_blocks, (nrec + BINB_TILE - 1) / BINB_TILE));
    const int64_t seg = ((nrec + G - 1) / G + BINB_TILE - 1) / BINB_TILE * BINB_TILE;
    k_binb_classify<<<G, BINB_WARPS * 32, 0, st>>>(b.rec, b.keys, nrec, seg, geo, b.hist);
    k_bin_rowscan<<<(ERI_NBINS + 1 + 7) / 8, 256, 0, st>>>(b.hist, G, total);
    k_bin_scan<<<1, 1024, 0, st>>>(total, b.dbounds);
    k_binb_scatter<<<G, BINB_WARPS * 32, 0, st>>>(b.rec, b.keys, nrec, seg, b.hist, b.dbounds, b.rec2);
    for (int k = 0; k < 4; ++k) note_launch();
    if (after_sort) cudaEventRecord(after_sort, st);
    e.rec = b.rec2;
    e.n = 0;
    e.dbounds = b.dbounds;
    // The 32 class kernels are independent (integer K / counter atomics) and each is a
    // persistent grid whose blocks finish within a few percent of one another: dealt over
    // several streams (st + helpers, forked and joined with events) the next kernel's blocks
    // fill the SMs a finishing kernel vacates instead of waiting for its last block.  That pays
    // while P and K fit L2 (c3 naive -2.9 %, c4 fourfold -0.9 % on the ERI kernels with 4
    // streams) and costs once they do not (c5 +1.9 %: classes running side by side dilute the
    // bra-major locality), so 4 streams up to 128 MB of P, else 1.  HXF_ERI_STREAMS overrides.
    static const int env_streams = [] {
        const char* v = getenv("HXF_ERI_STREAMS");
        return v ? std::max(1, std::min(4, atoi(v))) : 0;
    }();
    const int n_streams = env_streams ? env_streams
                          : ((int64_t)e.nfn * e.nfn * 8 <= (128ll << 20) && nrec >= (1 << 20) ? 4 : 1);
    EriStreams& xs = eri_streams();
    cudaStream_t lanes[4] = {st, st, st, st};
    if (n_streams > 1) {
        xs.ensure();
        HXF_CUDA(cudaEventRecord(xs.fork, st));
        for (int k = 1; k < n_streams; ++k) {
            lanes[k] = xs.s[k - 1];
            HXF_CUDA(cudaStreamWaitEvent(lanes[k], xs.fork, 0));
        }
    }
    // the heavy classes first, near and far alternating over the streams
    static const int order[16] = {0, 4, 1, 8, 2, 5, 12, 3, 9, 6, 10, 7, 13, 11, 14, 15};
    int slot = 0;
    for (int k = 0; k < 16; ++k) {
        launch_eri_class(order[k], false, e, lanes[slot++ % n_streams]);
        launch_eri_class(order[k], true, e, lanes[slot++ % n_streams]);
    }
    if (n_streams > 1)
        for (int k = 1; k < n_streams; ++k) {
            HXF_CUDA(cudaEventRecord(xs.join[k - 1], lanes[k]));
            HXF_CUDA(cudaStreamWaitEvent(st, xs.join[k - 1], 0));
        }
    HXF_CUDA(cudaGetLastError());
}

// the survivor buffers of one chunk set (cap records)
void survivor_bufs_alloc(SurvivorBufs& sb, int64_t cap, cudaStream_t st) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    sb.rec = lalloc<uint64_t>(cap, st);
    sb.rec2 = lalloc<uint64_t>(cap, st);
    sb.keys = lalloc<uint16_t>(cap, st);
    // 48 columns (blocks) per SM, 6 resident: a finer deal and more loads in flight measured
    // better up to here (8: 403 ms, 24: 346, 48: 334 per c5 build); HXF_BIN_BLOCKS=k overrides
    const char* bb = getenv("HXF_BIN_BLOCKS");
    sb.bin_blocks = sms * std::max(1, std::min(64, bb ? atoi(bb) : 48));
    sb.hist = lalloc<unsigned>((size_t)(ERI_NBINS + 1) * sb.bin_blocks, st);
    sb.dbounds = lalloc<int64_t>(2 * (ERI_NBINS + 2), st);   // bin starts, then the bin totals
}

void survivor_bufs_free(SurvivorBufs& sb, cudaStream_t st) {
    for (void* p : {(void*)sb.rec, (void*)sb.rec2, (void*)sb.keys, (void*)sb.hist, (void*)sb.dbounds})
        hxf_cache_free(p, st);
}

void host_ledger_add(unsigned long long* acc, const unsigned long long* v) {
    unsigned long long carry = 0;
    for (int k = 0; k < LEDGER_LIMBS; ++k) {
        unsigned long long s = acc[k] + v[k];
        unsigned long long c1 = s < acc[k];
        unsigned long long s2 = s + carry;
        unsigned long long c2 = s2 < s;
        acc[k] = s2;
        carry = c1 + c2;
    }
}

}  // namespace

// Per-build ERI pair tables: the pair records and sort-key bytes with each
// pair's primitive count cut to the primitives with S > thr (epp holds them
// first, sorted by S); at least one primitive is kept.
// finfo / fcnt: the same for the far-field kernels -- a collapsible pair (hxf_pairs::fcol)
// is the one point charge at epp[n_prim + pair id]; fcnt = far-field primitive count - 1,
// the sort-key nibble k_classify_far writes for a far quartet.
__global__ void k_prune_pairs(int64_t n, const int4* __restrict__ info, const uint8_t* __restrict__ meta,
                              const double* __restrict__ eS, double thr, int4* einfo, uint8_t* emeta,
                              const uint8_t* __restrict__ fcol, int64_t n_prim, int4* finfo, uint8_t* fcnt) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const int4 v = info[t];
    int keep = 0;
    while (keep < v.w && eS[v.z + keep] > thr) ++keep;
    keep = max(keep, 1);
    einfo[t] = make_int4(v.x, v.y, v.z, keep);
    emeta[t] = (uint8_t)((meta[t] & 3) | ((keep - 1) << 2));
    const bool col = fcol[t] != 0;
    finfo[t] = col ? make_int4(v.x, v.y, (int)(n_prim + t), 1) : make_int4(v.x, v.y, v.z, keep);
    fcnt[t] = (uint8_t)(col ? 0 : keep - 1);
}

struct EriTables {
    int4* info = nullptr;
    uint8_t* meta = nullptr;
    int4* finfo = nullptr;
    uint8_t* fcnt = nullptr;
};

// thr = HXF_PRIM_EPS / (max S of the other side * max|P|)
EriTables prune_tables(const hxf_pairs* pr, double other_smax, double pmax, cudaStream_t st) {
    EriTables t;
    t.info = lalloc<int4>(pr->n_pairs, st);
    t.meta = lalloc<uint8_t>(pr->n_pairs, st);
    t.finfo = lalloc<int4>(pr->n_pairs, st);
    t.fcnt = lalloc<uint8_t>(pr->n_pairs, st);
    // HXF_PRIM_EPS in the environment overrides the neglect threshold (0: keep every primitive);
    // a diagnostic hook for the tests, read per build
    const char* pe = getenv("HXF_PRIM_EPS");
    const double eps = pe ? atof(pe) : HXF_PRIM_EPS;
    const double thr = eps / (std::max(other_smax, 1e-300) * std::max(pmax, 1e-300));
    if (pr->n_pairs) {
        k_prune_pairs<<<(unsigned)((pr->n_pairs + 255) / 256), 256, 0, st>>>(pr->n_pairs, pr->info, pr->meta, pr->eS,
                                                                           thr, t.info, t.meta, pr->fcol,
                                                                           pr->n_prim_pairs, t.finfo, t.fcnt);
        note_launch();
    }
    return t;
}

void free_tables(EriTables& t, cudaStream_t st) {
    if (t.info) hxf_cache_free(t.info, st);
    if (t.meta) hxf_cache_free(t.meta, st);
    if (t.finfo) hxf_cache_free(t.finfo, st);
    if (t.fcnt) hxf_cache_free(t.fcnt, st);
    t = EriTables();
}

// Fixed-point scale of the K accumulator.  Any accumulator element (x, y)
// receives terms -1/2 P_uv (x u|v y) with |(x u|v y)| <= sqrt(Q_{s(x)s(u)})
// sqrt(Q_{s(v)s(y)}), each (x,u,v,y) at most 8 times over the symmetric
// images and slots, so sum |contributions| <= 1/2 * 8 * A_bra A_ket max|P|
// (A = hxf_pairs::amax).  S puts that bound below 2^61: partial sums never
// overflow the signed 64-bit accumulator.
int k_scale_bits(const hxf_pairs* bra, const hxf_pairs* ket, const hxf_density* dens) {
    const double B = 4.0 * std::max(bra->amax, 1e-300) * std::max(ket->amax, 1e-300) *
                     std::max(dens->maxabs, 1e-300) * (1.0 + 1e-9);
    int S = 61 - (int)std::ceil(std::log2(B));
    return std::max(-900, std::min(S, 900));
}

int fixed_to_double_impl(const int64_t* Kfx, int64_t n2, int S, double* K, cudaStream_t st) {
    if (n2 > 0) {
        k_fx_to_double<<<1024, 256, 0, st>>>(reinterpret_cast<const unsigned long long*>(Kfx), n2, S, K);
        note_launch();
    }
    HXF_CUDA(cudaGetLastError());
    return HXF_OK;
}

// A + A^T in place on a fixed-point accumulator (exact integer adds): the eightfold epilogue,
// and the symmetric form a shard's partial takes before a row-owning reduce-scatter
void fold_fixed_device(int64_t* K, int n, cudaStream_t st) {
    if (n <= 0) return;
    k_fold_fx<<<1024, 256, 0, st>>>(reinterpret_cast<unsigned long long*>(K), n);
    note_launch();
    HXF_CUDA(cudaGetLastError());
}

int hxf_last_timings_impl(double* ms, int n) {
    for (int k = 0; k < n && k < 8; ++k) ms[k] = g_timings[k];
    return HXF_OK;
}

// ---------------------------------------------------------------------------

int exchange_run(hxf_pairs* bra, hxf_pairs* ket, hxf_density* dens, const hxf_exchange_opts* o,
                 double* K_out, hxf_counters* out, cudaStream_t st) {
    NvtxRange nvtx_build("hxf: exchange build");
    hxf_system* s = bra->sys;
    if (ket->sys != s || dens->sys != s)
        throw HxfError{HXF_EINVAL, "bra, ket and P must be built over the same partition"};
    if (!(o->tau_2e >= 0.0)) throw HxfError{HXF_EINVAL, "tau_2e must be non-negative"};
    if (o->mode != HXF_MODE_SCHWARZ && o->mode != HXF_MODE_LITERAL)
        throw HxfError{HXF_EINVAL, "unknown screening mode"};
    if (o->symmetry != HXF_NAIVE && o->symmetry != HXF_FOURFOLD && o->symmetry != HXF_EIGHTFOLD)
        throw HxfError{HXF_EINVAL, "unknown symmetry driver"};
    if (o->symmetry != HXF_NAIVE && bra != ket)
        throw HxfError{HXF_EINVAL, "the fourfold driver takes a single pair tree"};
    for (int k = 0; k < 8; ++k) g_timings[k] = 0.0;
    Timer ttot(st);
    const int sym = o->symmetry != HXF_NAIVE;
    const int eight = o->symmetry == HXF_EIGHTFOLD;
    long long* dcount = lalloc<long long>(C_NCOUNTERS, st);
    unsigned long long* dledger = lalloc<unsigned long long>(LEDGER_LIMBS, st);
    HXF_CUDA(cudaMemsetAsync(dcount, 0, C_NCOUNTERS * sizeof(long long), st));
    HXF_CUDA(cudaMemsetAsync(dledger, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));

    // tie records (task and leaf stages): bounded device log, copied out at the end
    TieLog tl{nullptr, nullptr, 0};
    if (o->tie_log || o->tie_count) {
        tl.cap = o->tie_log ? std::max<int64_t>(o->tie_capacity, 0) : 0;
        tl.rec = lalloc<hxf_tie_record>(std::max<long long>(tl.cap, 1), st);
        tl.count = lalloc<unsigned long long>(1, st);
        HXF_CUDA(cudaMemsetAsync(tl.count, 0, sizeof(unsigned long long), st));
    }

    // ---- traversal
    Timer ttrav(st);
    TravInput ti{s, bra, ket, dens, o->tau_2e, o->mode, eight ? 2 : sym, o->shard_level, o->shard_begin,
                 o->shard_end, o->shard_stride, o->shard_mask, 0, 0, dcount, dledger};
    ti.root_level = o->root_level;
    ti.root_index = o->root_index;
    // a diagonal subtree start: K_out is the block of the start span's functions
    const bool subtree = o->root_level != 0 || o->root_index != 0;
    int64_t sub_f0 = 0, sub_n = s->nfn;
    if (subtree) {
        if (o->root_level < 0 || o->root_level >= s->n_levels || o->root_index < 0 ||
            o->root_index >= s->h_off[o->root_level + 1] - s->h_off[o->root_level])
            throw HxfError{HXF_EINVAL, "traversal start node outside the partition"};
        if (o->K_fixed) throw HxfError{HXF_EINVAL, "K_fixed requires the tree root as the start node"};
        const int k = s->h_off[o->root_level] + o->root_index;
        sub_f0 = s->h_flo[k];
        sub_n = s->h_fhi[k] - s->h_flo[k];
    }
    TraversalResult tr = traverse(ti, st);
    g_timings[0] = ttrav.stop();

    const int64_t n2 = (int64_t)s->nfn * s->nfn;
    long long hc[C_NCOUNTERS];
    unsigned long long hl[LEDGER_LIMBS];
    HXF_CUDA(cudaMemcpyAsync(hc, dcount, sizeof(hc), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaMemcpyAsync(hl, dledger, sizeof(hl), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    if (tl.count && hc[C_TIE_TASK] > 0) {
        // task-stage tie records: the traversal once more with the logging kernels
        // (counters and ledger into scratch); off the timed path of a tie-free build
        NvtxRange nvtx_ties("hxf: tie records (task stage)");
        long long* c2 = lalloc<long long>(C_NCOUNTERS, st);
        unsigned long long* l2 = lalloc<unsigned long long>(LEDGER_LIMBS, st);
        HXF_CUDA(cudaMemsetAsync(c2, 0, C_NCOUNTERS * sizeof(long long), st));
        HXF_CUDA(cudaMemsetAsync(l2, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
        TravInput t2 = ti;
        t2.counters = c2;
        t2.ledger = l2;
        t2.ties = tl;
        TraversalResult r2 = traverse(t2, st);
        for (void* p : {(void*)c2, (void*)l2, (void*)r2.leaf, (void*)r2.frontier})
            if (p) hxf_cache_free(p, st);
    }

    // Leaf tasks in bra-node-major order (stable radix sort on the bra leaf ids, bits 0-29 of
    // the task word; the traversal leaves them in the product tree's interleaved order): with
    // the screen's block-cyclic task runs, neighbouring survivor records share the bra node's
    // pair records, primitives, P rows and K rows.  Any order gives the same counters and,
    // through the integer accumulators, bitwise the same K and ledger words.
    {
        const char* ls = getenv("HXF_LEAF_SORT");
        const int leaf_sort = ls ? atoi(ls) : 1;
        if (leaf_sort && tr.n_leaf > 4096) {
            NvtxRange nvtx_ls("hxf: leaf task order");
            Timer tls(st);
            uint64_t* sorted = lalloc<uint64_t>(tr.n_leaf, st);
            size_t tb = 0;
            HXF_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, tr.leaf, sorted, tr.n_leaf, 0, 30, st));
            void* tmp = lalloc<char>(tb, st);
            HXF_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, tr.leaf, sorted, tr.n_leaf, 0, 30, st));
            note_launch();
            hxf_cache_free(tmp, st);
            hxf_cache_free(tr.leaf, st);
            tr.leaf = sorted;
            g_timings[0] += tls.stop();   // counted with the traversal
        }
    }
    ScreenArgs sa;
    sa.tasks = tr.leaf;
    const char* tb_env = getenv("HXF_TASK_BLOCK");
    const int tblock_max = std::max(1, tb_env ? atoi(tb_env) : 32);
    sa.tblock = 1;
    // HXF_SCREEN_DYN=0: the screen's task runs are dealt block-cyclically instead of handed out
    // by a device counter
    const char* dyn_env = getenv("HXF_SCREEN_DYN");
    const bool screen_dyn = dyn_env ? atoi(dyn_env) != 0 : true;
    unsigned* drun = lalloc<unsigned>(1, st);
    sa.next_run = nullptr;
    std::vector<int> lslo(s->n_leaves), lshi(s->n_leaves);
    {
        const int D = s->n_levels - 1;
        for (int k = s->h_off[D]; k < s->h_off[D + 1]; ++k) {
            lslo[s->h_leaf_id[k]] = s->h_slo[k];
            lshi[s->h_leaf_id[k]] = s->h_shi[k];
        }
    }
    int* d_lslo = lalloc<int>(s->n_leaves, st);
    int* d_lshi = lalloc<int>(s->n_leaves, st);
    HXF_CUDA(cudaMemcpyAsync(d_lslo, lslo.data(), lslo.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    HXF_CUDA(cudaMemcpyAsync(d_lshi, lshi.data(), lshi.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    sa.lslo = d_lslo;
    sa.lshi = d_lshi;
    sa.nleaf = s->n_leaves;
    sa.bra_base = bra->leaf_base;
    sa.ket_base = ket->leaf_base;
    sa.qb = bra->q;
    sa.qk = ket->q;
    sa.l = s->basis.l;
    sa.poff = s->basis.poff;
    sa.sqb = bra->sq;
    sa.sqk = ket->sq;
    // ERI pair tables of this build (negligible primitive tails dropped)
    EriTables etb = prune_tables(bra, ket->smax_prim, dens->maxabs, st);
    EriTables etk = bra == ket ? EriTables() : prune_tables(ket, bra->smax_prim, dens->maxabs, st);
    const EriTables& etk_use = bra == ket ? etb : etk;
    sa.metab = etb.meta;
    sa.metak = etk_use.meta;
    sa.pmax = dens->pmax;
    sa.ncidb = bra->ncid;
    sa.nvecb = bra->nvec;
    sa.nvecb_tri = bra->nvec_tri;
    sa.ncidk = ket->ncid;
    sa.nveck = ket->nvec;
    sa.nveck_tri = ket->nvec_tri;
    sa.ns = s->ns;
    sa.fn = s->basis.fn;
    sa.nf = s->basis.nf;
    sa.P = dens->P;
    sa.nfn = s->nfn;
    sa.tau = o->tau_2e;
    sa.mode = o->mode;
    sa.bpi = bra->pi;
    sa.bpj = bra->pj;
    sa.kpi = ket->pi;
    sa.kpj = ket->pj;
    sa.ties = tl;
    sa.n_bpairs = bra->n_pairs;
    sa.n_kpairs = ket->n_pairs;

    int dev_sms = 148;
    cudaDeviceGetAttribute(&dev_sms, cudaDevAttrMultiProcessorCount, s->device);
    // fixed grid (depends only on the device): the task -> warp assignment, and
    // so every per-warp ledger partial, is reproducible
    // HXF_SCREEN=flat selects the per-quartet screen (A/B reference)
    const char* sv = getenv("HXF_SCREEN");
    const bool flat = (sv && !strcmp(sv, "flat")) || s->max_leaf_shells > STAGED_MAXS;
    const bool ms8 = s->max_leaf_shells <= 8;
    const int sw = flat ? SCREEN_WARPS
                        : (ms8 ? (sym ? screen2_warps<true, 8>() : screen2_warps<false, 8>())
                               : (sym ? screen2_warps<true, 10>() : screen2_warps<false, 10>()));
    // 48 blocks per SM (4 are resident): the cost of a warp's task runs varies, and a finer
    // deal evens the tail of each chunk's launch (c5 screen: 12 -> 1818 ms, 24 -> 1755, 36 -> 1697,
    // 48 -> 1655, 96 -> 1734).  With the runs handed out dynamically (HXF_SCREEN_DYN, default) the
    // grid no longer matters (4 / 8 / 48: 1595 ms).  HXF_SCREEN_BLOCKS=k overrides.
    const char* sbk = getenv("HXF_SCREEN_BLOCKS");
    const int screen_per_sm = sbk ? std::max(1, atoi(sbk)) : (sym ? 48 : 32);
    const unsigned screen_grid = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((tr.n_leaf + sw - 1) / sw, (int64_t)dev_sms * screen_per_sm));
    auto launch_screen = [&](bool emit) {
        // task runs per warp: up to tblock_max, shorter when the range would leave warps idle
        sa.tblock = (int)std::max<int64_t>(1, std::min<int64_t>(tblock_max, (sa.t1 - sa.t0) / ((int64_t)screen_grid * sw)));
        sa.next_run = nullptr;
        if (screen_dyn && !flat) {
            cudaMemsetAsync(drun, 0, sizeof(unsigned), st);
            sa.next_run = drun;
        }
        if (flat) {
            if (eight) { if (emit) k_screen<true, true, true><<<screen_grid, sw * 32, 0, st>>>(sa); else k_screen<true, false, true><<<screen_grid, sw * 32, 0, st>>>(sa); }
            else if (sym) { if (emit) k_screen<true, true><<<screen_grid, sw * 32, 0, st>>>(sa); else k_screen<true, false><<<screen_grid, sw * 32, 0, st>>>(sa); }
            else { if (emit) k_screen<false, true><<<screen_grid, sw * 32, 0, st>>>(sa); else k_screen<false, false><<<screen_grid, sw * 32, 0, st>>>(sa); }
        } else {
            const dim3 g(screen_grid), b(sw * 32);
            if (ms8) {
                if (eight) { if (emit) k_screen2<true, true, 8, true><<<g, b, 0, st>>>(sa); else k_screen2<true, false, 8, true><<<g, b, 0, st>>>(sa); }
                else if (sym) { if (emit) k_screen2<true, true, 8><<<g, b, 0, st>>>(sa); else k_screen2<true, false, 8><<<g, b, 0, st>>>(sa); }
                else { if (emit) k_screen2<false, true, 8><<<g, b, 0, st>>>(sa); else k_screen2<false, false, 8><<<g, b, 0, st>>>(sa); }
            } else {
                if (eight) { if (emit) k_screen2<true, true, 10, true><<<g, b, 0, st>>>(sa); else k_screen2<true, false, 10, true><<<g, b, 0, st>>>(sa); }
                else if (sym) { if (emit) k_screen2<true, true, 10><<<g, b, 0, st>>>(sa); else k_screen2<true, false, 10><<<g, b, 0, st>>>(sa); }
                else { if (emit) k_screen2<false, true, 10><<<g, b, 0, st>>>(sa); else k_screen2<false, false, 10><<<g, b, 0, st>>>(sa); }
            }
        }
        note_launch();
    };

    const int S = k_scale_bits(bra, ket, dens);

    unsigned long long* Kfx = nullptr;
    int64_t logged = 0;
    int32_t* dlog = nullptr;
    unsigned long long* dlogfill = nullptr;
    const bool want_log = o->quartet_log != nullptr && o->evaluate;
    if (want_log) {
        dlog = lalloc<int32_t>(4 * std::max<int64_t>(o->log_capacity, 1), st);
        dlogfill = lalloc<unsigned long long>(1, st);
        HXF_CUDA(cudaMemsetAsync(dlogfill, 0, sizeof(unsigned long long), st));
    }

    unsigned long long* ddigest = nullptr;
    const bool want_digest = o->digest != nullptr && o->evaluate;
    if (want_digest) {
        ddigest = lalloc<unsigned long long>(3, st);
        HXF_CUDA(cudaMemsetAsync(ddigest, 0, 3 * sizeof(unsigned long long), st));
    }

    long long* scount = lalloc<long long>(C_NCOUNTERS, st);
    unsigned long long* sledger = lalloc<unsigned long long>(LEDGER_LIMBS, st);
    unsigned long long* dfill = lalloc<unsigned long long>(1, st);
    long long acc_c[C_NCOUNTERS];
    unsigned long long acc_l[LEDGER_LIMBS];
    memcpy(acc_c, hc, sizeof(acc_c));
    memcpy(acc_l, hl, sizeof(acc_l));

    if (!o->evaluate || tr.n_leaf == 0) {
        if (tr.n_leaf) {
            Timer tsc(st);
            HXF_CUDA(cudaMemsetAsync(scount, 0, C_NCOUNTERS * sizeof(long long), st));
            HXF_CUDA(cudaMemsetAsync(sledger, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
            sa.t0 = 0;
            sa.t1 = tr.n_leaf;
            sa.rec = nullptr;
            sa.cap = 0;
            sa.fill = dfill;
            sa.counters = scount;
            sa.ledger = sledger;
            launch_screen(false);
            HXF_CUDA(cudaGetLastError());
            long long c2[C_NCOUNTERS];
            unsigned long long l2[LEDGER_LIMBS];
            HXF_CUDA(cudaMemcpyAsync(c2, scount, sizeof(c2), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaMemcpyAsync(l2, sledger, sizeof(l2), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaStreamSynchronize(st));
            for (int k = 0; k < C_NCOUNTERS; ++k) acc_c[k] += c2[k];
            host_ledger_add(acc_l, l2);
            g_timings[1] = tsc.stop();
        }
    } else {
        Kfx = lalloc<unsigned long long>(n2, st);
        HXF_CUDA(cudaMemsetAsync(Kfx, 0, n2 * sizeof(unsigned long long), st));
        // HXF_PIPE=1 double-buffers the survivor chunks: the screen of chunk
        // i+1 (stream st) runs while chunk i is sorted and evaluated (stream
        // se).  Measured neutral (c5 -1%, c4 +5%): the persistent ERI kernels
        // fill every SM's registers, so the two stages cannot co-reside and
        // only the tails overlap.  Default: one buffer set, in order.
        const char* pv = getenv("HXF_PIPE");
        const bool pipe = pv && pv[0] == '1';
        const int NB = pipe ? 2 : 1;
        // (a full-size chunk set is 2^29 records x 160 B; when not even a quarter of that is free,
        // the cached scratch of other builds is handed back first)
        const size_t freeb = hxf_free_memory((size_t)160 * NB << 27);
        // survivor chunk capacity: ~40 B of device memory per record and buffer
        // set (two record buffers, two key buffers, radix-sort scratch)
        const int64_t cap = std::min<int64_t>(1ll << 29, std::max<int64_t>(1 << 16, (int64_t)(freeb / (160 * NB))));
        SurvivorBufs sb[2];
        unsigned long long* bfill[2];
        long long* bcount[2];
        unsigned long long* bledger[2];
        for (int b = 0; b < NB; ++b) {
            survivor_bufs_alloc(sb[b], cap, st);
            sb[b].bgeo = bra->geo;
            sb[b].kgeo = ket->geo;
            sb[b].bgip = bra->gip;
            sb[b].kgip = ket->gip;
            sb[b].bfcnt = etb.fcnt;
            sb[b].kfcnt = etk_use.fcnt;
            bfill[b] = b == 0 ? dfill : lalloc<unsigned long long>(1, st);
            bcount[b] = b == 0 ? scount : lalloc<long long>(C_NCOUNTERS, st);
            bledger[b] = b == 0 ? sledger : lalloc<unsigned long long>(LEDGER_LIMBS, st);
        }
        // ERI-side counters (primitive / class counts) accumulate over all chunks
        long long* ecount = lalloc<long long>(C_NCOUNTERS, st);
        HXF_CUDA(cudaMemsetAsync(ecount, 0, C_NCOUNTERS * sizeof(long long), st));
        EriArgs e;
        e.dbounds = nullptr;
        e.bpi = bra->pi;
        e.bpj = bra->pj;
        e.bppoff = bra->ppoff;
        e.bpp = bra->epp;
        e.kpi = ket->pi;
        e.kpj = ket->pj;
        e.kppoff = ket->ppoff;
        e.kpp = ket->epp;
        e.binfo = etb.info;
        e.kinfo = etk_use.info;
        e.bfinfo = etb.finfo;
        e.kfinfo = etk_use.finfo;
        e.ctr = s->basis.ctr;
        e.fn = s->basis.fn;
        e.P = dens->P;
        e.nfn = s->nfn;
        e.S = S;
        e.K = Kfx;
        e.counters = ecount;
        e.n_bpairs = bra->n_pairs;
        e.n_kpairs = ket->n_pairs;
        e.n_bprim = bra->n_prim_pairs + bra->n_pairs;
        e.n_kprim = ket->n_prim_pairs + ket->n_pairs;
        cudaStream_t se = st;
        cudaEvent_t ev_in = nullptr, ev_scr[2] = {nullptr, nullptr}, ev_eri[2] = {nullptr, nullptr};
        if (pipe) {
            // the ERI stream yields SM slots to the screen whenever blocks retire
            int lo_prio = 0, hi_prio = 0;
            cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
            const char* pr = getenv("HXF_PIPE_PRIO");
            HXF_CUDA(cudaStreamCreateWithPriority(&se, cudaStreamNonBlocking, (pr && pr[0] == '0') ? 0 : lo_prio));
            HXF_CUDA(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
            for (int b = 0; b < 2; ++b) {
                HXF_CUDA(cudaEventCreateWithFlags(&ev_scr[b], cudaEventDisableTiming));
                HXF_CUDA(cudaEventCreateWithFlags(&ev_eri[b], cudaEventDisableTiming));
            }
            HXF_CUDA(cudaEventRecord(ev_in, st));   // Kfx / counters zeroed before any ERI
            HXF_CUDA(cudaStreamWaitEvent(se, ev_in, 0));
        }
        std::vector<std::pair<cudaEvent_t, cudaEvent_t>> eri_ev;
        std::vector<cudaEvent_t> sort_ev;   // after classification + sort + key bounds, per chunk
        bool used[2] = {false, false};
        int cur = 0;
        int64_t chunk = std::max<int64_t>(1, cap / 1024);
        int64_t t0 = 0;
        while (t0 < tr.n_leaf) {
            const int64_t t1 = std::min(tr.n_leaf, t0 + chunk);
            // the buffer set must be free: the ERI work that last read it is done
            if (pipe && used[cur]) HXF_CUDA(cudaStreamWaitEvent(st, ev_eri[cur], 0));
            Timer tsc(st);
            HXF_CUDA(cudaMemsetAsync(bcount[cur], 0, C_NCOUNTERS * sizeof(long long), st));
            HXF_CUDA(cudaMemsetAsync(bledger[cur], 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
            HXF_CUDA(cudaMemsetAsync(bfill[cur], 0, sizeof(unsigned long long), st));
            sa.t0 = t0;
            sa.t1 = t1;
            sa.rec = sb[cur].rec;
            sa.keys = sb[cur].keys;
            sa.cap = cap;
            sa.fill = bfill[cur];
            sa.counters = bcount[cur];
            sa.ledger = bledger[cur];
            nvtxRangePushA("hxf: leaf screen");
            launch_screen(true);
            nvtxRangePop();
            HXF_CUDA(cudaGetLastError());
            unsigned long long fill = 0;
            long long c2[C_NCOUNTERS];
            unsigned long long l2[LEDGER_LIMBS];
            HXF_CUDA(cudaMemcpyAsync(&fill, bfill[cur], sizeof(fill), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaMemcpyAsync(c2, bcount[cur], sizeof(c2), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaMemcpyAsync(l2, bledger[cur], sizeof(l2), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaStreamSynchronize(st));
            g_timings[1] += tsc.stop();
            if ((int64_t)fill > cap) {
                if (t1 - t0 == 1) throw HxfError{HXF_ELOGIC, "survivor buffer too small for one leaf task"};
                chunk = std::max<int64_t>(1, (t1 - t0) / 2);
                continue;
            }
            for (int k = 0; k < C_NCOUNTERS; ++k) acc_c[k] += c2[k];
            host_ledger_add(acc_l, l2);
            const int64_t nrec = (int64_t)fill;
            if (nrec) {
                cudaEvent_t ea, eb;
                cudaEventCreate(&ea);
                cudaEventCreate(&eb);
                if (pipe) {
                    HXF_CUDA(cudaEventRecord(ev_scr[cur], st));
                    HXF_CUDA(cudaStreamWaitEvent(se, ev_scr[cur], 0));
                }
                cudaEvent_t es;
                cudaEventCreate(&es);
                HXF_CUDA(cudaEventRecord(ea, se));
                nvtxRangePushA("hxf: ERI stage");
                eri_sorted_stage_async(e, sb[cur], nrec, se, es);
                nvtxRangePop();
                HXF_CUDA(cudaEventRecord(eb, se));
                eri_ev.push_back({ea, eb});
                sort_ev.push_back(es);
                if (want_log)
                    { k_log<<<(unsigned)((nrec + 255) / 256), 256, 0, se>>>(sb[cur].rec2, nrec, bra->pi, bra->pj, ket->pi,
                                                                        ket->pj, dlog, o->log_capacity, dlogfill); note_launch(); }
                if (want_digest)
                    { k_digest<<<(unsigned)std::min<int64_t>((nrec + 255) / 256, 4096), 256, 0, se>>>(
                          sb[cur].rec2, nrec, bra->pi, bra->pj, ket->pi, ket->pj, (uint64_t)s->ns, o->digest_mod,
                          o->digest_rem, eight, ddigest); note_launch(); }
                if (pipe) {
                    HXF_CUDA(cudaEventRecord(ev_eri[cur], se));
                    used[cur] = true;
                }
            }
            const double dens_per_task = (double)nrec / (double)(t1 - t0);
            chunk = std::max<int64_t>(1, (int64_t)(0.85 * cap / std::max(dens_per_task, 1.0)));
            t0 = t1;
            if (pipe) cur ^= 1;
        }
        if (pipe) {
            // the epilogue (stream st) follows every ERI launch
            HXF_CUDA(cudaEventRecord(ev_in, se));
            HXF_CUDA(cudaStreamWaitEvent(st, ev_in, 0));
        }
        HXF_CUDA(cudaStreamSynchronize(se));
        for (size_t k = 0; k < eri_ev.size(); ++k) {
            float ms = 0.f, ms_sort = 0.f;
            cudaEventElapsedTime(&ms, eri_ev[k].first, eri_ev[k].second);
            cudaEventElapsedTime(&ms_sort, eri_ev[k].first, sort_ev[k]);
            g_timings[2] += ms;             // the whole ERI stage
            g_timings[5] += ms - ms_sort;   // ERI + contraction kernels only
            g_timings[6] += ms_sort;        // far-field classification + sort + key bounds
            cudaEventDestroy(eri_ev[k].first);
            cudaEventDestroy(eri_ev[k].second);
            cudaEventDestroy(sort_ev[k]);
        }
        long long ce[C_NCOUNTERS];
        HXF_CUDA(cudaMemcpyAsync(ce, ecount, sizeof(ce), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        for (int k = 0; k < C_NCOUNTERS; ++k) acc_c[k] += ce[k];
        if (pipe) {
            cudaEventDestroy(ev_in);
            for (int b = 0; b < 2; ++b) {
                cudaEventDestroy(ev_scr[b]);
                cudaEventDestroy(ev_eri[b]);
            }
            cudaStreamDestroy(se);
        }
        for (int b = 0; b < NB; ++b) {
            survivor_bufs_free(sb[b], st);
            if (b) {
                hxf_cache_free(bfill[b], st);
                hxf_cache_free(bcount[b], st);
                hxf_cache_free(bledger[b], st);
            }
        }
        hxf_cache_free(ecount, st);
    }

    if (o->count_screen_bytes && tr.n_leaf) {
        HXF_CUDA(cudaMemsetAsync(scount, 0, C_NCOUNTERS * sizeof(long long), st));
        k_screen_bytes<<<(unsigned)std::min<int64_t>((tr.n_leaf + 255) / 256, (int64_t)dev_sms * 16), 256, 0, st>>>(
            tr.leaf, tr.n_leaf, d_lslo, d_lshi, sym, scount);
        note_launch();
        long long c2[C_NCOUNTERS];
        HXF_CUDA(cudaMemcpyAsync(c2, scount, sizeof(c2), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        acc_c[C_SCREEN_BYTES] = c2[C_SCREEN_BYTES];
    }
    if (tl.count && acc_c[C_TIE_LEAF] > 0 && tr.n_leaf) {
        // leaf-stage tie records: the per-quartet screen once more over every leaf task
        // with the logging instantiation (no emission, counters and ledger into scratch)
        NvtxRange nvtx_ties("hxf: tie records (leaf stage)");
        HXF_CUDA(cudaMemsetAsync(scount, 0, C_NCOUNTERS * sizeof(long long), st));
        HXF_CUDA(cudaMemsetAsync(sledger, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
        sa.t0 = 0;
        sa.t1 = tr.n_leaf;
        sa.rec = nullptr;
        sa.keys = nullptr;
        sa.cap = 0;
        sa.fill = dfill;
        sa.counters = scount;
        sa.ledger = sledger;
        const unsigned g = (unsigned)std::max<int64_t>(
            1, std::min<int64_t>((tr.n_leaf + SCREEN_WARPS - 1) / SCREEN_WARPS, (int64_t)dev_sms * 8));
        if (eight) k_screen<true, false, true, true><<<g, SCREEN_WARPS * 32, 0, st>>>(sa);
        else if (sym) k_screen<true, false, false, true><<<g, SCREEN_WARPS * 32, 0, st>>>(sa);
        else k_screen<false, false, false, true><<<g, SCREEN_WARPS * 32, 0, st>>>(sa);
        note_launch();
        HXF_CUDA(cudaGetLastError());
    }

    // ---- epilogue
    NvtxRange nvtx_epilogue("hxf: epilogue");
    Timer tep(st);
    if (eight && Kfx) {  // K = A + A^T, exact in fixed point (each |entry| < 2^61)
        k_fold_fx<<<1024, 256, 0, st>>>(Kfx, s->nfn);
        note_launch();
    }
    if (K_out && o->K_fixed) {
        if (!o->K_on_device) throw HxfError{HXF_EINVAL, "K_fixed requires K_on_device"};
        if (Kfx) HXF_CUDA(cudaMemcpyAsync(K_out, Kfx, n2 * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, st));
        else HXF_CUDA(cudaMemsetAsync(K_out, 0, n2 * sizeof(unsigned long long), st));
        if (o->K_scale) *o->K_scale = S;
    } else if (K_out) {
        double* Kd = (o->K_on_device && !subtree) ? K_out : lalloc<double>(n2, st);
        if (Kfx) {
            { k_fx_to_double<<<1024, 256, 0, st>>>(Kfx, n2, S, Kd); note_launch(); }
            if (sym && !eight && o->symmetrize) {
                unsigned long long* dm = lalloc<unsigned long long>(1, st);
                HXF_CUDA(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
                { k_asym<<<1024, 256, 0, st>>>(Kd, s->nfn, dm); note_launch(); }
                unsigned long long hm = 0;
                HXF_CUDA(cudaMemcpyAsync(&hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, st));
                HXF_CUDA(cudaStreamSynchronize(st));
                hxf_cache_free(dm, st);
                double asym;
                memcpy(&asym, &hm, sizeof(asym));
                if (asym > 1e-10) {
                    char buf[160];
                    snprintf(buf, sizeof(buf), "asymmetry %.3e exceeds 1.0e-10; symmetry update set is inconsistent", asym);
                    throw HxfError{HXF_ELOGIC, buf};
                }
                { k_symmetrize<<<1024, 256, 0, st>>>(Kd, s->nfn); note_launch(); }
            }
        } else {
            HXF_CUDA(cudaMemsetAsync(Kd, 0, n2 * sizeof(double), st));
        }
        if (subtree) {  // the start span's block, local indices
            HXF_CUDA(cudaMemcpy2DAsync(K_out, sub_n * sizeof(double), Kd + sub_f0 * s->nfn + sub_f0,
                                       s->nfn * sizeof(double), sub_n * sizeof(double), sub_n,
                                       o->K_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
            hxf_cache_free(Kd, st);
        } else if (!o->K_on_device) {
            xfer_to_host(K_out, Kd, n2 * sizeof(double), st);
            hxf_cache_free(Kd, st);
        }
    }
    if (want_log) {
        unsigned long long lf = 0;
        HXF_CUDA(cudaMemcpyAsync(&lf, dlogfill, sizeof(lf), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        logged = (int64_t)lf;
        const int64_t ncopy = std::min<int64_t>(logged, o->log_capacity);
        if (ncopy) HXF_CUDA(cudaMemcpyAsync(o->quartet_log, dlog, 4 * ncopy * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        hxf_cache_free(dlog, st);
        hxf_cache_free(dlogfill, st);
    }
    if (o->log_count) *o->log_count = logged;
    if (tl.count) {
        unsigned long long nt = 0;
        HXF_CUDA(cudaMemcpyAsync(&nt, tl.count, sizeof(nt), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        const int64_t ncopy = std::min<int64_t>((int64_t)nt, tl.cap);
        if (ncopy) HXF_CUDA(cudaMemcpyAsync(o->tie_log, tl.rec, ncopy * sizeof(hxf_tie_record), cudaMemcpyDeviceToHost, st));
        if (o->tie_count) *o->tie_count = (int64_t)nt;
        HXF_CUDA(cudaStreamSynchronize(st));
        hxf_cache_free(tl.rec, st);
        hxf_cache_free(tl.count, st);
    }
    if (o->digest) {
        unsigned long long hd[3] = {0, 0, 0};
        if (want_digest) {
            HXF_CUDA(cudaMemcpyAsync(hd, ddigest, sizeof(hd), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaStreamSynchronize(st));
            hxf_cache_free(ddigest, st);
        }
        for (int k = 0; k < 3; ++k) o->digest[k] = hd[k];
    }
    for (void* p : {(void*)Kfx, (void*)scount, (void*)sledger, (void*)dfill, (void*)dcount,
                    (void*)dledger, (void*)d_lslo, (void*)d_lshi, (void*)tr.leaf, (void*)drun})
        if (p) hxf_cache_free(p, st);
    free_tables(etb, st);
    free_tables(etk, st);
    HXF_CUDA(cudaStreamSynchronize(st));
    HXF_CUDA(cudaGetLastError());
    g_timings[3] = tep.stop();
    g_timings[4] = ttot.stop();

    // ---- counters out
    hxf_counters& c = *out;
    c.tasks_visited = acc_c[C_VISITED];
    c.tasks_culled_screening = acc_c[C_CULL_SCREEN];
    c.tasks_culled_absent = acc_c[C_CULL_ABSENT];
    c.leaf_contractions = acc_c[C_LEAF];
    c.eri_shell_quartets = acc_c[C_ERIQ];
    c.quartets_culled_leaf = acc_c[C_CULL_LEAF];
    c.tasks_expanded = acc_c[C_EXPANDED];
    c.children_spawned = acc_c[C_SPAWNED];
    c.links_culled_screening = acc_c[C_LINK_SCREEN];
    c.links_culled_absent = acc_c[C_LINK_ABSENT];
    for (int k = 0; k < HXF_NCASES; ++k) {
        c.case_tasks[k] = acc_c[C_CASE0 + k];
        c.case_leaf_tasks[k] = acc_c[C_CASELEAF0 + k];
    }
    c.ties_task = acc_c[C_TIE_TASK];
    c.ties_leaf = acc_c[C_TIE_LEAF];
    c.screen_bytes = acc_c[C_SCREEN_BYTES];
    c.prim_quartets = acc_c[C_PRIMQ];
    for (int k = 0; k < 16; ++k) {
        c.class_quartets[k] = acc_c[C_CLSQ0 + k];
        c.class_prim_quartets[k] = acc_c[C_CLSPQ0 + k];
    }
    c.culled_bound_ledger = fx_to_double<LEDGER_LIMBS>(acc_l, LEDGER_SCALE);
    if (acc_c[C_OVERFLOW]) throw HxfError{HXF_ELOGIC, "device bounds check failed (HXF_DEBUG_BOUNDS build)"};
    static const bool eri_stats = getenv("HXF_ERI_STATS") != nullptr;
    if (eri_stats)
        fprintf(stderr, "eri: quartets %lld far %lld (%.1f%%), primitive quartets %lld far %lld (%.1f%%)\n",
                acc_c[C_ERIQ], acc_c[C_DBG0], 100.0 * acc_c[C_DBG0] / std::max(1ll, acc_c[C_ERIQ]),
                acc_c[C_PRIMQ], acc_c[C_DBG0 + 1], 100.0 * acc_c[C_DBG0 + 1] / std::max(1ll, acc_c[C_PRIMQ]));
#ifdef HXF_PROF_SCREEN
    fprintf(stderr, "screen cycles (warp-summed): staging %.3e tables %.3e phase1 %.3e phase2 %.3e\n",
            (double)acc_c[C_DBG0], (double)acc_c[C_DBG0 + 1], (double)acc_c[C_DBG0 + 2],
            (double)acc_c[C_DBG0 + 3]);
    fprintf(stderr, "screen tasks %lld: cell-test culled %lld, zero survivors %lld\n", acc_c[C_DBG0 + 5],
            acc_c[C_DBG0 + 4], acc_c[C_DBG0 + 6]);
#endif
    return HXF_OK;
}

// ---------------------------------------------------------------------------
// Direct-SCF twin (the semantics of dense_exchange_screened,
// oracle.py:69-108): every ordered shell quartet (i,j,k,l) of live pairs with
// (f(Q_ij) |P|_jk) f(Q_kl) > tau, found without the hierarchy, evaluated by
// the same sorted ERI stage into the same fixed-point K.  Because the K
// accumulation is order-independent, the twin's K equals the hierarchical
// naive K bit for bit exactly when both evaluate the same quartet set: the
// full-size K parity check of SURVEY.md 8(c) item 2.
//
// Enumeration: per shell j the ket rows k sorted by |P|_jk descending, per
// shell k the columns l sorted by f(Q_kl) descending (segmented radix sorts
// of the dense n_shells^2 tables); one warp per bra pair walks its k list 32
// at a time, each lane binary-searches the passing prefix of its l list
// (binary64 products are monotone), and the walk stops at the first k whose
// bound with max f(Q) cannot pass.  A count pass and an exclusive scan give
// every bra pair its record range, so the emit pass writes without atomics.

namespace {

__global__ void k_direct_tables(int64_t n_pairs, const int* pi, const int* pj, const double* q,
                                const double* sq, int schwarz, int ns, double* fq, int* pidm) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n_pairs) return;
    const int64_t x = (int64_t)pi[t] * ns + pj[t];
    fq[x] = schwarz ? sq[t] : q[t];
    pidm[x] = (int)t;
}

__global__ void k_iota_cols(int64_t n2, int ns, int* col, int64_t* row_off) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t < n2) col[t] = (int)(t % ns);
    if (t <= ns) row_off[t] = t * ns;
}

// entries > 0 per row of a row-wise descending-sorted table
__global__ void k_row_nnz(const double* sorted, int ns, int* cnt) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= ns) return;
    const double* row = sorted + (int64_t)r * ns;
    int lo = 0, hi = ns;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (row[mid] > 0.0) lo = mid + 1;
        else hi = mid;
    }
    cnt[r] = lo;
}

struct DirectArgs {
    int64_t n_pairs;
    const int* pi;
    const int* pj;
    const uint8_t* meta;
    const double* fq;   // n_shells^2, f(Q), 0 where absent
    const int* pidm;    // n_shells^2, pair id, -1 where absent
    const double* pm;   // n_shells^2, block max |P|
    const int* lq;      // per k: l sorted by f(Q_kl) descending
    const int* nq;
    const int* lp;      // per j: k sorted by |P|_jk descending
    const int* np;
    int ns;
    int mod, rem;
    double tau, fqmax;
    int64_t* count;        // count pass: records per bra pair
    const int64_t* off;    // emit pass: record offsets (exclusive scan of count)
    uint64_t* rec;
    uint16_t* keys;
};

template <bool EMIT>
__global__ void __launch_bounds__(256) k_direct(DirectArgs a, int64_t p0, int64_t p1) {
    const int lane = threadIdx.x & 31;
    const int64_t p = p0 + (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32;
    if (p >= p1) return;
    const int ia = a.pi[p], ib = a.pj[p];
    int64_t wcount = 0;
    if (a.mod <= 1 || ia % a.mod == a.rem) {
        const int64_t ns = a.ns;
        const double fab = a.fq[ia * ns + ib];
        const int* krow = a.lp + ib * ns;
        const int nk = a.np[ib];
        const int ca = a.meta[p];
        const int64_t base = EMIT ? a.off[p] - a.off[p0] : 0;
        for (int c0 = 0; c0 < nk; c0 += 32) {
            const int idx = c0 + lane;
            int k = -1, n = 0;
            double x = 0.0;
            bool stop = idx >= nk;
            if (!stop) {
                k = krow[idx];
                x = __dmul_rn(fab, a.pm[ib * ns + k]);
                if (!(__dmul_rn(x, a.fqmax) > a.tau)) {
                    stop = true;
                    k = -1;
                }
            }
            const int* lrow = a.lq + (int64_t)(k < 0 ? 0 : k) * ns;
            if (k >= 0) {
                int lo = 0, hi = a.nq[k];
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (__dmul_rn(x, a.fq[(int64_t)k * ns + lrow[mid]]) > a.tau) lo = mid + 1;
                    else hi = mid;
                }
                n = lo;
            }
            int incl = n;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += v;
            }
            if (EMIT) {
                int64_t pos = base + wcount + incl - n;
                for (int t = 0; t < n; ++t, ++pos) {
                    const int pk = a.pidm[(int64_t)k * ns + lrow[t]];
                    const int cb = a.meta[pk];
                    const uint64_t cls = (uint64_t)(((ca & 3) << 2) | (cb & 3));
                    a.rec[pos] = (uint64_t)p | ((uint64_t)pk << 28) | (1ull << 56);
                    a.keys[pos] = (uint16_t)((cls << 8) | ((ca >> 2) << 4) | (cb >> 2));
                }
            }
            wcount += __shfl_sync(0xffffffffu, incl, 31);
            if (__any_sync(0xffffffffu, stop)) break;
        }
    }
    if (!EMIT && lane == 0) a.count[p] = wcount;
}

}  // namespace

int direct_run(hxf_pairs* pairs, hxf_density* dens, const hxf_exchange_opts* o, double* K_out,
               hxf_counters* out, cudaStream_t st) {
    NvtxRange nvtx_build("hxf: direct twin");
    hxf_system* s = pairs->sys;
    if (dens->sys != s) throw HxfError{HXF_EINVAL, "pairs and P must be built over the same partition"};
    if (!(o->tau_2e >= 0.0)) throw HxfError{HXF_EINVAL, "tau_2e must be non-negative"};
    if (o->mode != HXF_MODE_SCHWARZ && o->mode != HXF_MODE_LITERAL)
        throw HxfError{HXF_EINVAL, "unknown screening mode"};
    for (int k = 0; k < 8; ++k) g_timings[k] = 0.0;
    Timer ttot(st);
    const int ns = s->ns;
    const int64_t n2 = (int64_t)ns * ns, nfn2 = (int64_t)s->nfn * s->nfn;
    const int schwarz = o->mode == HXF_MODE_SCHWARZ;
    const int mod = std::max(1, o->digest_mod), rem = o->digest_rem;

    // ---- dense f(Q) / pair-id tables and the two row-sorted lists
    Timer tprep(st);
    double* fq = lalloc<double>(n2, st);
    int* pidm = lalloc<int>(n2, st);
    HXF_CUDA(cudaMemsetAsync(fq, 0, n2 * sizeof(double), st));
    HXF_CUDA(cudaMemsetAsync(pidm, 0xff, n2 * sizeof(int), st));
    { k_direct_tables<<<(unsigned)((pairs->n_pairs + 255) / 256), 256, 0, st>>>(
          pairs->n_pairs, pairs->pi, pairs->pj, pairs->q, pairs->sq, schwarz, ns, fq, pidm); note_launch(); }
    int* iota = lalloc<int>(n2, st);
    int64_t* roff = lalloc<int64_t>(ns + 1, st);
    { k_iota_cols<<<(unsigned)((std::max<int64_t>(n2, ns + 1) + 255) / 256), 256, 0, st>>>(n2, ns, iota, roff); note_launch(); }
    double* skeys = lalloc<double>(n2, st);
    int* lq = lalloc<int>(n2, st);
    int* lp = lalloc<int>(n2, st);
    int* nq = lalloc<int>(ns, st);
    int* np = lalloc<int>(ns, st);
    size_t tb = 0;
    HXF_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(nullptr, tb, fq, skeys, iota, lq, n2, ns, roff, roff + 1, 0, 64, st));
    void* stmp = lalloc<char>(tb, st);
    size_t tb2 = tb;
    HXF_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(stmp, tb2, fq, skeys, iota, lq, n2, ns, roff, roff + 1, 0, 64, st));
    { k_row_nnz<<<(ns + 255) / 256, 256, 0, st>>>(skeys, ns, nq); note_launch(); }
    tb2 = tb;
    HXF_CUDA(cub::DeviceSegmentedRadixSort::SortPairsDescending(stmp, tb2, dens->pmax, skeys, iota, lp, n2, ns, roff, roff + 1, 0, 64, st));
    { k_row_nnz<<<(ns + 255) / 256, 256, 0, st>>>(skeys, ns, np); note_launch(); }
    HXF_CUDA(cudaGetLastError());
    for (void* p : {(void*)stmp, (void*)skeys, (void*)iota, (void*)roff}) hxf_cache_free(p, st);

    DirectArgs da;
    da.n_pairs = pairs->n_pairs;
    da.pi = pairs->pi;
    da.pj = pairs->pj;
    EriTables et = prune_tables(pairs, pairs->smax_prim, dens->maxabs, st);
    da.meta = et.meta;
    da.fq = fq;
    da.pidm = pidm;
    da.pm = dens->pmax;
    da.lq = lq;
    da.nq = nq;
    da.lp = lp;
    da.np = np;
    da.ns = ns;
    da.mod = mod;
    da.rem = rem;
    da.tau = o->tau_2e;
    da.fqmax = schwarz ? std::sqrt(pairs->maxq) : pairs->maxq;
    // ---- count pass + offsets
    const int64_t npr = pairs->n_pairs;
    int64_t* cnt = lalloc<int64_t>(npr + 1, st);
    int64_t* off = lalloc<int64_t>(npr + 1, st);
    HXF_CUDA(cudaMemsetAsync(cnt + npr, 0, sizeof(int64_t), st));
    da.count = cnt;
    da.off = nullptr;
    da.rec = nullptr;
    da.keys = nullptr;
    const unsigned grid_all = (unsigned)((npr * 32 + 255) / 256);
    if (npr) { k_direct<false><<<grid_all, 256, 0, st>>>(da, 0, npr); note_launch(); }
    size_t stb = 0;
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, stb, cnt, off, npr + 1, st));
    void* scan_tmp = lalloc<char>(stb, st);
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp, stb, cnt, off, npr + 1, st));
    std::vector<int64_t> hoff(npr + 1);
    HXF_CUDA(cudaMemcpyAsync(hoff.data(), off, (npr + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    hxf_cache_free(scan_tmp, st);
    hxf_cache_free(cnt, st);
    g_timings[0] = tprep.stop();
    const int64_t total = hoff[npr];

    // ---- fixed-point K (the hierarchical build's scale: bitwise-comparable K)
    const int S = k_scale_bits(pairs, pairs, dens);
    unsigned long long* Kfx = nullptr;
    long long* scount = lalloc<long long>(C_NCOUNTERS, st);
    HXF_CUDA(cudaMemsetAsync(scount, 0, C_NCOUNTERS * sizeof(long long), st));
    unsigned long long* ddigest = nullptr;
    const bool want_digest = o->digest != nullptr && o->evaluate;
    if (want_digest) {
        ddigest = lalloc<unsigned long long>(3, st);
        HXF_CUDA(cudaMemsetAsync(ddigest, 0, 3 * sizeof(unsigned long long), st));
    }
    if (o->evaluate && total) {
        Kfx = lalloc<unsigned long long>(nfn2, st);
        HXF_CUDA(cudaMemsetAsync(Kfx, 0, nfn2 * sizeof(unsigned long long), st));
        const size_t freeb = hxf_free_memory((size_t)160 << 27);
        const int64_t cap = std::min<int64_t>(1ll << 29, std::max<int64_t>(1 << 16, (int64_t)(freeb / 160)));
        SurvivorBufs sb;
        survivor_bufs_alloc(sb, cap, st);
        sb.bgeo = sb.kgeo = pairs->geo;   // the same far-field decisions as the hierarchical drivers
        sb.bgip = sb.kgip = pairs->gip;
        sb.bfcnt = sb.kfcnt = et.fcnt;
        EriArgs e;
        e.dbounds = nullptr;
        e.bpi = e.kpi = pairs->pi;
        e.bpj = e.kpj = pairs->pj;
        e.bppoff = e.kppoff = pairs->ppoff;
        e.bpp = e.kpp = pairs->epp;
        e.binfo = e.kinfo = et.info;
        e.bfinfo = e.kfinfo = et.finfo;
        e.ctr = s->basis.ctr;
        e.fn = s->basis.fn;
        e.P = dens->P;
        e.nfn = s->nfn;
        e.S = S;
        e.K = Kfx;
        e.counters = scount;
        e.n_bpairs = e.n_kpairs = pairs->n_pairs;
        e.n_bprim = e.n_kprim = pairs->n_prim_pairs + pairs->n_pairs;
        da.off = off;
        da.rec = sb.rec;
        da.keys = sb.keys;
        int64_t p0 = 0;
        while (p0 < npr) {
            // largest p1 with hoff[p1] - hoff[p0] <= cap
            int64_t p1 = std::upper_bound(hoff.begin() + p0 + 1, hoff.end(), hoff[p0] + cap) - hoff.begin() - 1;
            if (p1 <= p0) throw HxfError{HXF_ELOGIC, "survivor buffer too small for one bra pair"};
            const int64_t nrec = hoff[p1] - hoff[p0];
            if (nrec) {
                Timer tsc(st);
                { k_direct<true><<<(unsigned)(((p1 - p0) * 32 + 255) / 256), 256, 0, st>>>(da, p0, p1); note_launch(); }
                g_timings[1] += tsc.stop();
                Timer teri(st);
                eri_sorted_stage_async(e, sb, nrec, st);
                if (want_digest)
                    { k_digest<<<(unsigned)std::min<int64_t>((nrec + 255) / 256, 4096), 256, 0, st>>>(
                          sb.rec2, nrec, pairs->pi, pairs->pj, pairs->pi, pairs->pj, (uint64_t)ns, mod, rem, 0,
                          ddigest); note_launch(); }
                HXF_CUDA(cudaStreamSynchronize(st));
                g_timings[2] += teri.stop();
            }
            p0 = p1;
        }
        survivor_bufs_free(sb, st);
    }
    // ---- epilogue
    Timer tep(st);
    if (K_out) {
        double* Kd = o->K_on_device ? K_out : lalloc<double>(nfn2, st);
        if (Kfx) { k_fx_to_double<<<1024, 256, 0, st>>>(Kfx, nfn2, S, Kd); note_launch(); }
        else HXF_CUDA(cudaMemsetAsync(Kd, 0, nfn2 * sizeof(double), st));
        if (!o->K_on_device) {
            xfer_to_host(K_out, Kd, nfn2 * sizeof(double), st);
            hxf_cache_free(Kd, st);
        }
    }
    long long hc[C_NCOUNTERS];
    HXF_CUDA(cudaMemcpyAsync(hc, scount, sizeof(hc), cudaMemcpyDeviceToHost, st));
    unsigned long long hd[3] = {0, 0, 0};
    if (want_digest) HXF_CUDA(cudaMemcpyAsync(hd, ddigest, sizeof(hd), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    if (o->digest)
        for (int k = 0; k < 3; ++k) o->digest[k] = hd[k];
    for (void* p : {(void*)Kfx, (void*)scount, (void*)ddigest, (void*)fq, (void*)pidm, (void*)lq, (void*)lp,
                    (void*)nq, (void*)np, (void*)off})
        if (p) hxf_cache_free(p, st);
    free_tables(et, st);
    HXF_CUDA(cudaStreamSynchronize(st));
    HXF_CUDA(cudaGetLastError());
    g_timings[3] = tep.stop();
    g_timings[4] = ttot.stop();
    hxf_counters& c = *out;
    memset(&c, 0, sizeof(c));
    c.eri_shell_quartets = total;
    c.prim_quartets = hc[C_PRIMQ];
    for (int k = 0; k < 16; ++k) {
        c.class_quartets[k] = hc[C_CLSQ0 + k];
        c.class_prim_quartets[k] = hc[C_CLSPQ0 + k];
    }
    return HXF_OK;
}

// ---------------------------------------------------------------------------
// utilities exported through the C ABI

namespace {
__global__ void k_dfma(double* out, int iters) {
    double a0 = threadIdx.x * 1e-9, a1 = a0 + 1e-9, a2 = a0 + 2e-9, a3 = a0 + 3e-9;
    double a4 = a0 + 4e-9, a5 = a0 + 5e-9, a6 = a0 + 6e-9, a7 = a0 + 7e-9;
    const double b = 0.999999999, c = 1e-12;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
            a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
        }
    }
    const double s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == 12345.0) out[0] = s;  // keep the chain alive
}
}  // namespace

int symmetrize_device(double* K, int n, double tol, cudaStream_t st) {
    unsigned long long* dm = lalloc<unsigned long long>(1, st);
    HXF_CUDA(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
    { k_asym<<<1024, 256, 0, st>>>(K, n, dm); note_launch(); }
    unsigned long long hm = 0;
    HXF_CUDA(cudaMemcpyAsync(&hm, dm, sizeof(hm), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    hxf_cache_free(dm, st);
    double asym;
    memcpy(&asym, &hm, sizeof(asym));
    if (asym > tol) {
        char buf[160];
        snprintf(buf, sizeof(buf), "asymmetry %.3e exceeds %.1e; symmetry update set is inconsistent", asym, tol);
        throw HxfError{HXF_ELOGIC, buf};
    }
    { k_symmetrize<<<1024, 256, 0, st>>>(K, n); note_launch(); }
    HXF_CUDA(cudaGetLastError());
    return HXF_OK;
}

double fp64_peak(cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = lalloc<double>(1, st);
    const int iters = 2048, threads = 512, blocks = sms * 4;
    { k_dfma<<<blocks, threads, 0, st>>>(out, 16); note_launch(); }  // warm-up
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    { k_dfma<<<blocks, threads, 0, st>>>(out, iters); note_launch(); }
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    hxf_cache_free(out, st);
    HXF_CUDA(cudaGetLastError());
    const double flops = 2.0 * 8 * 16 * (double)iters * threads * blocks;
    return flops / (ms * 1e-3) / 1e12;
}

int frontier_run(hxf_pairs* bra, hxf_pairs* ket, hxf_density* dens, double tau, int mode, int sym,
                 int level, int64_t* n_tasks, double* cost, int64_t cap, cudaStream_t st) {
    hxf_system* s = bra->sys;
    long long* dcount = lalloc<long long>(C_NCOUNTERS, st);
    unsigned long long* dledger = lalloc<unsigned long long>(LEDGER_LIMBS, st);
    HXF_CUDA(cudaMemsetAsync(dcount, 0, C_NCOUNTERS * sizeof(long long), st));
    HXF_CUDA(cudaMemsetAsync(dledger, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
    TravInput ti{s, bra, ket, dens, tau, mode, sym, -1, 0, 0, 1, nullptr, 1, level, dcount, dledger};
    TraversalResult tr = traverse(ti, st);
    *n_tasks = tr.n_frontier;
    if (cost) {
        const int64_t n = std::min<int64_t>(cap, tr.n_frontier);
        for (int64_t k = 0; k < n; ++k) cost[k] = 1.0;
    }
    for (void* p : {(void*)dcount, (void*)dledger, (void*)tr.leaf, (void*)tr.frontier})
        if (p) hxf_cache_free(p, st);
    HXF_CUDA(cudaStreamSynchronize(st));
    return HXF_OK;
}
