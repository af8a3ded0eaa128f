// Level-synchronous product-tree traversal (SURVEY.md kernels K4/K5).
//
// Restates the reference's recursive visitors as a breadth-first expansion:
//   naive      exchange_naive.py:124-154   task (bra, P, ket) = spans (mu,nu,lam,sig)
//   symmetric  exchange_symmetry.py:233-294 task (bra, ket, 4 density refs, alive)
// Every expanded task of level L spawns its (up to 16) children; each child is
// visited (absent / screened / leaf / expand) by one thread, and survivors are
// compacted with a block-wide scan into the next frontier or the leaf-task
// list.  Compaction is two-pass (count, device scan, write), so frontiers and
// per-block partial sums are in a deterministic order and repeated builds are
// bitwise identical (the reference's determinism contract,
// test_exchange_naive.py:157-162).
//
// Task encoding (uint64): four 15-bit span indices (level-local for frontier
// tasks, partition-leaf ids for leaf tasks) and a 4-bit live-slot mask.

#include <cub/cub.cuh>

#include "hxf_internal.cuh"
#include "traverse.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace {
// HXF_TRAV_TRACE=1: per-level host timestamps on stderr (diagnostic only)
inline double trav_now_ms() {
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
}  // namespace

#define TRAV_STRIPES 1024

namespace {

enum { O_NONE = 0, O_ABSENT, O_SCREEN, O_LEAF, O_EXPAND };
enum { CASE_A = 0, CASE_B, CASE_C, CASE_D, CASE_E, CASE_F1, CASE_F2, CASE_H, CASE_SPARSE };

struct LevelView {
    int n;                 // spans at this level
    int64_t node_off;      // offset of this level's dense node arrays
    const int* leaf_id;    // per span (level-local pointer)
    const int* flo;
    int level;             // partition level (tie records)
};

// bf / kf: the task factors f(norm) (sqrt(norm) for Schwarz, norm for literal),
// negative where pruned; b/k row, col: sqrt of the row / column sum maxima
struct TreeView {
    const double* bf;
    const double* brow;
    const double* bcol;
    const double* kf;
    const double* krow;
    const double* kcol;
    const double* pnorm;
    double tau;
    int mode;
    TieLog ties;
};

struct Visit {
    int outcome;
    int live;
    int label;
    int links_screen;
    int links_absent;
    int tie;
    double ledger;
};


__device__ __forceinline__ bool is_tie(double bound, double tau) {
    return tau > 0.0 && fabs(bound - tau) <= 1e-12 * tau;
}

// culled_task_bound (exchange_naive.py:91-102); sbs / sks: the precomputed
// sqrt(max(rowsum or colsum, 0)) of the bra / ket node
__device__ __forceinline__ double ledger_term(double pn, double sbs, double sks) {
    return __dmul_rn(__dmul_rn(__dmul_rn(0.5, pn), sbs), sks);
}

// TIES: the diagnostic instantiation that also appends tie records (run a second time,
// only when a build counted ties and the caller asked for the log: the timed path has none)
template <bool TIES>
__device__ Visit visit_naive(const TreeView& tv, const LevelView& lv, int mu, int nu, int lam,
                             int sig) {
    Visit v{O_NONE, 0, 0, 0, 0, 0, 0.0};
    const int64_t n = lv.n;
    const int64_t ib = lv.node_off + mu * n + nu;
    const int64_t ip = lv.node_off + nu * n + lam;
    const int64_t ik = lv.node_off + lam * n + sig;
    const double fb = tv.bf[ib], np = tv.pnorm[ip], fk = tv.kf[ik];
    if (fb < 0.0 || np < 0.0 || fk < 0.0) {
        v.outcome = O_ABSENT;
        return v;
    }
    const double bound = sorted_product3(fb, np, fk);
    v.tie = is_tie(bound, tv.tau);
    if (TIES && v.tie) tie_emit(tv.ties, HXF_TIE_TASK, lv.level, 0, bound > tv.tau, mu, nu, lam, sig, bound, tv.tau);
    if (bound <= tv.tau) {
        v.outcome = O_SCREEN;
        v.ledger = ledger_term(np, tv.brow[ib], tv.kcol[ik]);
        return v;
    }
    const bool leaf = lv.leaf_id[mu] >= 0 && lv.leaf_id[nu] >= 0 && lv.leaf_id[lam] >= 0 &&
                      lv.leaf_id[sig] >= 0;
    v.outcome = leaf ? O_LEAF : O_EXPAND;
    v.live = 1;
    return v;
}

// _case_label (exchange_symmetry.py:135-173), span identity = index equality
__device__ __forceinline__ int case_label(const LevelView& lv, int mu, int nu, int lam, int sig) {
    if (mu == lam && nu == sig) return CASE_E;
    const bool bd = mu == nu, kd = lam == sig;
    if (bd && kd) return CASE_H;
    if (bd || kd) return CASE_B;
    if (nu == lam || mu == sig) return CASE_A;
    if (mu == lam) return CASE_F1;
    if (nu == sig) return CASE_F2;
    const int fmu = lv.flo[mu], fnu = lv.flo[nu], flam = lv.flo[lam], fsig = lv.flo[sig];
    if (fnu < flam || fsig < fmu) return CASE_A;
    if ((flam < fmu) != (fsig < fnu)) return CASE_C;
    return CASE_D;
}

template <bool TIES>
__device__ Visit visit_sym(const TreeView& tv, const LevelView& lv, int mu, int nu, int lam, int sig,
                           int alive) {
    Visit v{O_NONE, 0, 0, 0, 0, 0, 0.0};
    const int64_t n = lv.n;
    const int64_t ib = lv.node_off + mu * n + nu;
    const int64_t ik = lv.node_off + lam * n + sig;
    const double fb = tv.bf[ib], fk = tv.kf[ik];
    if (fb < 0.0 || fk < 0.0) {
        v.outcome = O_ABSENT;
        return v;
    }
    // slot refs: g0 P[nu,lam], g1 P[mu,lam], g2 P[nu,sig], g3 P[mu,sig]
    const int rr[4] = {nu, mu, nu, mu}, rc[4] = {lam, lam, sig, sig};
    bool screened = false, absent = false;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
        if (!((alive >> g) & 1)) continue;
        const double pn = tv.pnorm[lv.node_off + rr[g] * n + rc[g]];
        if (pn < 0.0) {
            v.links_absent++;
            absent = true;
            continue;
        }
        const double bound = sorted_product3(fb, pn, fk);
        if (is_tie(bound, tv.tau)) {
            ++v.tie;
            if (TIES) tie_emit(tv.ties, HXF_TIE_TASK, lv.level, g, bound > tv.tau, mu, nu, lam, sig, bound, tv.tau);
        }
        if (bound <= tv.tau) {
            v.links_screen++;
            screened = true;
            // _SLOT_TRANSPOSES (exchange_symmetry.py:53): g1, g3 transpose bra; g2, g3 ket
            const double bs = (g & 1) ? tv.bcol[ib] : tv.brow[ib];
            const double ks = (g & 2) ? tv.krow[ik] : tv.kcol[ik];
            v.ledger += ledger_term(pn, bs, ks);
            continue;
        }
        v.live |= 1 << g;
    }
    if (!v.live) {
        v.outcome = screened ? O_SCREEN : O_ABSENT;
        return v;
    }
    v.label = absent ? CASE_SPARSE : case_label(lv, mu, nu, lam, sig);
    const bool leaf = lv.leaf_id[mu] >= 0 && lv.leaf_id[nu] >= 0 && lv.leaf_id[lam] >= 0 &&
                      lv.leaf_id[sig] >= 0;
    v.outcome = leaf ? O_LEAF : O_EXPAND;
    return v;
}

__device__ __forceinline__ uint64_t pack_task(int a, int b, int c, int d, int live) {
    return (uint64_t)a | ((uint64_t)b << 15) | ((uint64_t)c << 30) | ((uint64_t)d << 45) |
           ((uint64_t)live << 60);
}

struct ExpandArgs {
    const uint64_t* in;
    int64_t n_in;
    const int* kid0;   // level-L spans (level-local pointers)
    const int* kid1;
    LevelView child;   // level L+1
    TreeView tv;
    uint64_t* out_expand;
    uint64_t* out_leaf;
    int* blk_counts;   // pass 1: per block packed (leaf | expand << 16)
    const int64_t* blk_off_expand;
    const int64_t* blk_off_leaf;
    long long* counters;
    unsigned long long* ledger;
    int eight;         // eightfold: children of a bra == ket task keep (bra) <= (ket)
    uint8_t* outc;     // per child thread: is_leaf | is_expand << 1 | live << 2 (count pass -> write pass)
};

// children of a span (a leaf stands in for itself, quadtree.py:47-49)
__device__ __forceinline__ int kids(const ExpandArgs& a, int s, int* k) {
    k[0] = a.kid0[s];
    k[1] = a.kid1[s];
    return k[1] < 0 ? 1 : 2;
}

// canonical child keys (exchange_symmetry.py:212-217)
__device__ __forceinline__ bool canon_key(int key, int r, int c, int nr, int nc, int* x, int* y) {
    if (r == c) {
        if (nr == 1) {
            *x = 0;
            *y = 0;
            return key == 0;
        }
        const int tx[3] = {0, 0, 1}, ty[3] = {0, 1, 1};
        if (key >= 3) return false;
        *x = tx[key];
        *y = ty[key];
        return true;
    }
    if (key >= nr * nc) return false;
    *x = key / nc;
    *y = key % nc;
    return true;
}

// Two passes per level.  Count pass: visit every child (norm gathers, bounds,
// counters, ledger), store a one-byte outcome per child and the block's leaf /
// expand counts.  Write pass: re-read the outcome byte (no second visit), scan,
// write the children's task words at their deterministic positions.
template <bool SYM>
__device__ __forceinline__ bool child_spans(const ExpandArgs& a, uint64_t task, int c, int* cm, int* cn,
                                            int* cl, int* cs) {
    const int mu = task & 0x7fff, nu = (task >> 15) & 0x7fff, lam = (task >> 30) & 0x7fff,
              sig = (task >> 45) & 0x7fff;
    int km[2], kn[2], kl[2], ks[2];
    const int nm = kids(a, mu, km), nn = kids(a, nu, kn), nl = kids(a, lam, kl), ns = kids(a, sig, ks);
    bool valid;
    if (!SYM) {
        const int ia = (c >> 3) & 1, ic = (c >> 2) & 1, id = (c >> 1) & 1, ibb = c & 1;
        valid = ia < nm && ic < nn && id < nl && ibb < ns;
        if (valid) {
            *cm = km[ia];
            *cn = kn[ic];
            *cl = kl[id];
            *cs = ks[ibb];
        }
    } else {
        int x, y, z, w;
        valid = canon_key(c >> 2, mu, nu, nm, nn, &x, &y) && canon_key(c & 3, lam, sig, nl, ns, &z, &w);
        if (valid) {
            *cm = km[x];
            *cn = kn[y];
            *cl = kl[z];
            *cs = ks[w];
            // eightfold: a task with bra node == ket node spawns each mirror pair
            // of children once (bra child <= ket child); tasks with bra < ket
            // keep every child (their mirrors live under the excluded mirror task)
            if (a.eight && mu == lam && nu == sig) valid = *cm < *cl || (*cm == *cl && *cn <= *cs);
        }
    }
    return valid;
}

// per-warp sum of 6-bit (or 8-bit) packed per-thread counts: one reduction per word
template <int N>
__device__ __forceinline__ void flush_packed(long long* counters, unsigned word, int bits, const int (&slots)[N]) {
    const unsigned s = __reduce_add_sync(0xffffffffu, word);
    if ((threadIdx.x & 31) == 0 && s) {
        const unsigned m = (1u << bits) - 1u;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            const unsigned v = (s >> (bits * k)) & m;
            if (v) atomic_add_ll(&counters[slots[k]], (long long)v);
        }
    }
}

template <bool SYM, bool WRITE, bool TIES = false>
__global__ void __launch_bounds__(256) k_expand(ExpandArgs a) {
    typedef cub::BlockScan<int, 256> Scan;
    typedef cub::BlockReduce<double, 256> Red;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Red::TempStorage red;
    } tmp;
    const int64_t t = blockIdx.x * 256ll + threadIdx.x;
    const int64_t parent = t >> 4;
    const int c = (int)(t & 15);
    if (WRITE) {
        const int oc = parent < a.n_in ? a.outc[t] : 0;
        const int is_leaf = oc & 1, is_exp = (oc >> 1) & 1, live = oc >> 2;
        int packed = is_leaf | (is_exp << 16), excl, total;
        Scan(tmp.scan).ExclusiveSum(packed, excl, total);
        if (is_leaf | is_exp) {
            int cm = 0, cn = 0, cl = 0, cs = 0;
            child_spans<SYM>(a, a.in[parent], c, &cm, &cn, &cl, &cs);
            if (is_leaf) {
                const int lid[4] = {a.child.leaf_id[cm], a.child.leaf_id[cn], a.child.leaf_id[cl], a.child.leaf_id[cs]};
                a.out_leaf[a.blk_off_leaf[blockIdx.x] + (excl & 0xffff)] = pack_task(lid[0], lid[1], lid[2], lid[3], live);
            } else {
                a.out_expand[a.blk_off_expand[blockIdx.x] + (excl >> 16)] = pack_task(cm, cn, cl, cs, live);
            }
        }
        return;
    }
    Visit v{O_NONE, 0, 0, 0, 0, 0, 0.0};
    if (parent < a.n_in) {
        const uint64_t task = a.in[parent];
        int cm = 0, cn = 0, cl = 0, cs = 0;
        if (child_spans<SYM>(a, task, c, &cm, &cn, &cl, &cs))
            v = SYM ? visit_sym<TIES>(a.tv, a.child, cm, cn, cl, cs, (int)(task >> 60))
                    : visit_naive<TIES>(a.tv, a.child, cm, cn, cl, cs);
        const int is_leaf = v.outcome == O_LEAF, is_exp = v.outcome == O_EXPAND;
        a.outc[t] = (uint8_t)(is_leaf | (is_exp << 1) | ((is_leaf | is_exp) ? (v.live << 2) : 0));
    }
    const int is_leaf = v.outcome == O_LEAF, is_exp = v.outcome == O_EXPAND;
    int packed = is_leaf | (is_exp << 16), excl, total;
    Scan(tmp.scan).ExclusiveSum(packed, excl, total);
    if (threadIdx.x == 0) a.blk_counts[blockIdx.x] = total;
    // counters: per-warp sums of packed per-thread counts, warp-aggregated
    // integer atomics (order independent) into one of TRAV_STRIPES copies, so
    // the ~10^8 warps of a deep level do not all serialise on the same addresses;
    // k_fold_stripes sums the copies
    long long* counters = a.counters + (blockIdx.x % TRAV_STRIPES) * C_NCOUNTERS;
    unsigned long long* ledger = a.ledger + (blockIdx.x % TRAV_STRIPES) * LEDGER_LIMBS;
    const unsigned valid_child = v.outcome != O_NONE;
    {
        const unsigned w0 = valid_child | (valid_child << 6) | ((unsigned)(v.outcome == O_SCREEN) << 12) |
                            ((unsigned)(v.outcome == O_ABSENT) << 18) | ((unsigned)is_leaf << 24);
        const int s0[5] = {C_VISITED, C_SPAWNED, C_CULL_SCREEN, C_CULL_ABSENT, C_LEAF};
        flush_packed(counters, w0, 6, s0);
        const unsigned w1 = (unsigned)is_exp | ((unsigned)v.tie << 8) | ((unsigned)v.links_screen << 16) |
                            ((unsigned)v.links_absent << 24);
        const int s1[4] = {C_EXPANDED, C_TIE_TASK, C_LINK_SCREEN, C_LINK_ABSENT};
        flush_packed(counters, w1, 8, s1);
    }
    if (SYM) {
        const unsigned counted = (unsigned)(is_leaf || is_exp);
        const unsigned lab = (unsigned)v.label;
        // one-hot label fields: labels 0-4 in one word, 5-8 in the next
        const unsigned c_lo = lab < 5 ? counted << (6 * lab) : 0u, c_hi = lab >= 5 ? counted << (6 * (lab - 5)) : 0u;
        const unsigned l_lo = lab < 5 ? (unsigned)is_leaf << (6 * lab) : 0u,
                       l_hi = lab >= 5 ? (unsigned)is_leaf << (6 * (lab - 5)) : 0u;
        const int sc0[5] = {C_CASE0, C_CASE0 + 1, C_CASE0 + 2, C_CASE0 + 3, C_CASE0 + 4};
        const int sc1[4] = {C_CASE0 + 5, C_CASE0 + 6, C_CASE0 + 7, C_CASE0 + 8};
        const int sl0[5] = {C_CASELEAF0, C_CASELEAF0 + 1, C_CASELEAF0 + 2, C_CASELEAF0 + 3, C_CASELEAF0 + 4};
        const int sl1[4] = {C_CASELEAF0 + 5, C_CASELEAF0 + 6, C_CASELEAF0 + 7, C_CASELEAF0 + 8};
        flush_packed(counters, c_lo, 6, sc0);
        flush_packed(counters, c_hi, 6, sc1);
        flush_packed(counters, l_lo, 6, sl0);
        flush_packed(counters, l_hi, 6, sl1);
    }
    __syncthreads();
    const double lsum = Red(tmp.red).Sum(v.ledger);
    if (threadIdx.x == 0 && lsum != 0.0) {
        unsigned long long limb[LEDGER_LIMBS];
        fx_from_double<LEDGER_LIMBS>(lsum, LEDGER_SCALE, limb);
        fx_atomic_add<LEDGER_LIMBS>(ledger, limb);
    }
}

// sum the striped counter / ledger copies into the real ones (one block)
__global__ void k_fold_stripes(const long long* sc, const unsigned long long* sl, long long* counters,
                               unsigned long long* ledger) {
    for (int k = threadIdx.x; k < C_NCOUNTERS; k += blockDim.x) {
        long long s = 0;
        for (int r = 0; r < TRAV_STRIPES; ++r) s += sc[r * C_NCOUNTERS + k];
        counters[k] += s;
    }
    if (threadIdx.x == 0) {
        for (int r = 0; r < TRAV_STRIPES; ++r) {
            unsigned long long carry = 0;
            for (int k = 0; k < LEDGER_LIMBS; ++k) {
                const unsigned long long a0 = ledger[k], b = sl[r * LEDGER_LIMBS + k];
                const unsigned long long t = a0 + b;
                const unsigned long long c1 = t < a0;
                const unsigned long long t2 = t + carry;
                const unsigned long long c2 = t2 < t;
                ledger[k] = t2;
                carry = c1 + c2;
            }
        }
    }
}

// the start task: the diagonal node (r, r) of the start level visited against
// itself (the root, or a diagonal subtree the caller passed as bra = ket = P)
template <bool SYM, bool TIES = false>
__global__ void k_root(TreeView tv, LevelView lv, int r, uint64_t* out_expand, uint64_t* out_leaf,
                       int* outcome, long long* counters, unsigned long long* ledger) {
    Visit v = SYM ? visit_sym<TIES>(tv, lv, r, r, r, r, 0xf) : visit_naive<TIES>(tv, lv, r, r, r, r);
    counters[C_VISITED] += 1;
    counters[C_CULL_SCREEN] += v.outcome == O_SCREEN;
    counters[C_CULL_ABSENT] += v.outcome == O_ABSENT;
    counters[C_LEAF] += v.outcome == O_LEAF;
    counters[C_EXPANDED] += v.outcome == O_EXPAND;
    counters[C_TIE_TASK] += v.tie;
    counters[C_LINK_SCREEN] += v.links_screen;
    counters[C_LINK_ABSENT] += v.links_absent;
    if (SYM && (v.outcome == O_LEAF || v.outcome == O_EXPAND)) {
        counters[C_CASE0 + v.label] += 1;
        if (v.outcome == O_LEAF) counters[C_CASELEAF0 + v.label] += 1;
    }
    if (v.ledger != 0.0) {
        unsigned long long limb[LEDGER_LIMBS];
        fx_from_double<LEDGER_LIMBS>(v.ledger, LEDGER_SCALE, limb);
        fx_atomic_add<LEDGER_LIMBS>(ledger, limb);
    }
    if (v.outcome == O_EXPAND) out_expand[0] = pack_task(r, r, r, r, v.live);
    if (v.outcome == O_LEAF)
        out_leaf[0] = pack_task(lv.leaf_id[r], lv.leaf_id[r], lv.leaf_id[r], lv.leaf_id[r], v.live);
    *outcome = v.outcome;
}

template <typename T>
T* talloc(size_t n, cudaStream_t st) {
    if (n == 0) n = 1;
    return (T*)hxf_cache_alloc(n * sizeof(T), st);
}

__global__ void k_unpack_counts(const int* packed, int64_t n, int64_t* leaf, int64_t* expand) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    leaf[t] = packed[t] & 0xffff;
    expand[t] = packed[t] >> 16;
}

}  // namespace

// Run the traversal.  Returns the leaf-task list (device, caller frees with
// hxf_cache_free).  Counters / ledger are accumulated into the device arrays.
// If shard_level >= 0 the expand frontier at that level is restricted to
// [shard_begin, shard_end) (every shard_stride-th task) and, unless shard_begin == 0, counters and leaf
// tasks produced above the cut are discarded (they belong to rank 0).
TraversalResult traverse(const TravInput& in, cudaStream_t st) {
    NvtxRange nvtx_range("hxf: traversal");
    hxf_system* s = in.sys;
    const bool schwarz = in.mode == HXF_MODE_SCHWARZ;
    TreeView tv{schwarz ? in.bra->snorm : in.bra->norm, in.bra->srow, in.bra->scol,
                schwarz ? in.ket->snorm : in.ket->norm, in.ket->srow, in.ket->scol, in.dens->norm, in.tau, in.mode,
                in.ties};
    TraversalResult res;
    res.leaf = nullptr;
    res.n_leaf = 0;
    res.frontier_sizes.clear();
    long long* counters = in.counters;
    unsigned long long* ledger = in.ledger;
    // discard counters above a shard cut on non-zero shards: accumulate into scratch
    long long* scratch_c = nullptr;
    unsigned long long* scratch_l = nullptr;
    const bool sharded = in.shard_level >= 0;
    const bool discard_top = sharded && in.shard_begin != 0;
    if (discard_top) {
        scratch_c = talloc<long long>(C_NCOUNTERS, st);
        scratch_l = talloc<unsigned long long>(LEDGER_LIMBS, st);
        HXF_CUDA(cudaMemsetAsync(scratch_c, 0, C_NCOUNTERS * sizeof(long long), st));
        HXF_CUDA(cudaMemsetAsync(scratch_l, 0, LEDGER_LIMBS * sizeof(unsigned long long), st));
        counters = scratch_c;
        ledger = scratch_l;
    }
    // striped copies of the counters / ledger for the expand kernels
    long long* sc = talloc<long long>((size_t)TRAV_STRIPES * C_NCOUNTERS, st);
    unsigned long long* sl = talloc<unsigned long long>((size_t)TRAV_STRIPES * LEDGER_LIMBS, st);
    auto zero_stripes = [&]() {
        HXF_CUDA(cudaMemsetAsync(sc, 0, sizeof(long long) * TRAV_STRIPES * C_NCOUNTERS, st));
        HXF_CUDA(cudaMemsetAsync(sl, 0, sizeof(unsigned long long) * TRAV_STRIPES * LEDGER_LIMBS, st));
    };
    auto fold_stripes = [&](long long* c, unsigned long long* l) {
        k_fold_stripes<<<1, 128, 0, st>>>(sc, sl, c, l);
        note_launch();
        zero_stripes();
    };
    zero_stripes();
    const int D = s->n_levels - 1;
    const int L0 = in.root_level;
    if (L0 < 0 || L0 > D || in.root_index < 0 || in.root_index >= s->h_off[L0 + 1] - s->h_off[L0])
        throw HxfError{HXF_EINVAL, "traversal start node outside the partition"};
    std::vector<uint64_t*> leaf_parts;
    std::vector<int64_t> leaf_counts;
    uint64_t* cur = talloc<uint64_t>(1, st);
    uint64_t* leaf0 = talloc<uint64_t>(1, st);
    int* d_outcome = talloc<int>(1, st);
    LevelView lv0{s->h_off[L0 + 1] - s->h_off[L0], s->node_off[L0], s->lv.leaf_id + s->h_off[L0],
                  s->lv.flo + s->h_off[L0], L0};
    const int r0 = in.root_index;
    const bool log_ties = in.ties.count != nullptr;   // the diagnostic pass (tie records)
    if (log_ties) {
        if (in.sym) { k_root<true, true><<<1, 1, 0, st>>>(tv, lv0, r0, cur, leaf0, d_outcome, counters, ledger); note_launch(); }
        else { k_root<false, true><<<1, 1, 0, st>>>(tv, lv0, r0, cur, leaf0, d_outcome, counters, ledger); note_launch(); }
    } else if (in.sym) { k_root<true><<<1, 1, 0, st>>>(tv, lv0, r0, cur, leaf0, d_outcome, counters, ledger); note_launch(); }
    else { k_root<false><<<1, 1, 0, st>>>(tv, lv0, r0, cur, leaf0, d_outcome, counters, ledger); note_launch(); }
    int outcome = 0;
    HXF_CUDA(cudaMemcpyAsync(&outcome, d_outcome, sizeof(int), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    hxf_cache_free(d_outcome, st);
    int64_t n_cur = outcome == O_EXPAND ? 1 : 0;
    if (outcome == O_LEAF) {
        leaf_parts.push_back(leaf0);
        leaf_counts.push_back(1);
    } else {
        hxf_cache_free(leaf0, st);
    }
    res.frontier_sizes.push_back(n_cur);
    bool cut_reached = false;
    for (int L = L0; L < D && n_cur > 0; ++L) {
        if (sharded && L == in.shard_level) {
            cut_reached = true;
            // restrict the frontier to this shard; from here on counters are real
            int64_t cnt = 0;
            uint64_t* part = nullptr;
            if (in.shard_mask) {  // arbitrary selection: order-preserving compaction by the mask
                const int64_t nm = std::min<int64_t>(std::max<int64_t>(in.shard_end, 0), n_cur);
                part = talloc<uint64_t>(std::max<int64_t>(nm, 1), st);
                if (nm > 0) {
                    uint8_t* dm = talloc<uint8_t>(nm, st);
                    int64_t* dn = talloc<int64_t>(1, st);
                    HXF_CUDA(cudaMemcpyAsync(dm, in.shard_mask, nm, cudaMemcpyHostToDevice, st));
                    size_t tb = 0;
                    HXF_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, cur, dm, part, dn, nm, st));
                    char* tmp = talloc<char>(tb, st);
                    HXF_CUDA(cub::DeviceSelect::Flagged(tmp, tb, cur, dm, part, dn, nm, st));
                    HXF_CUDA(cudaMemcpyAsync(&cnt, dn, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
                    HXF_CUDA(cudaStreamSynchronize(st));
                    for (void* p : {(void*)dm, (void*)dn, (void*)tmp}) hxf_cache_free(p, st);
                }
            } else {
                const int64_t b = std::min<int64_t>(in.shard_begin, n_cur);
                const int64_t e = std::min<int64_t>(std::max<int64_t>(in.shard_end, b), n_cur);
                const int64_t stride = std::max<int64_t>(in.shard_stride, 1);
                cnt = (e - b + stride - 1) / stride;
                part = talloc<uint64_t>(std::max<int64_t>(cnt, 1), st);
                if (cnt > 0)  // every stride-th task: a 2D copy of 8-byte rows
                    HXF_CUDA(cudaMemcpy2DAsync(part, sizeof(uint64_t), cur + b, stride * sizeof(uint64_t),
                                               sizeof(uint64_t), cnt, cudaMemcpyDeviceToDevice, st));
            }
            hxf_cache_free(cur, st);
            cur = part;
            n_cur = cnt;
            if (discard_top) {
                // leaf tasks above the cut belong to shard 0
                for (uint64_t* p : leaf_parts) hxf_cache_free(p, st);
                leaf_parts.clear();
                leaf_counts.clear();
            }
            fold_stripes(counters, ledger);  // above the cut: scratch (discarded) on shards != 0
            counters = in.counters;
            ledger = in.ledger;
            if (n_cur == 0) break;
        }
        if (in.frontier_only && L == in.frontier_level) break;
        const int n_par = s->h_off[L + 1] - s->h_off[L];
        (void)n_par;
        const int base_ch = s->h_off[L + 1];
        LevelView ch{s->h_off[L + 2] - s->h_off[L + 1], s->node_off[L + 1], s->lv.leaf_id + base_ch,
                     s->lv.flo + base_ch, L + 1};
        static const bool trace = getenv("HXF_TRAV_TRACE") != nullptr;
        const double tr0 = trace ? trav_now_ms() : 0.0;
        const int64_t nthreads = n_cur * 16;
        const int64_t nb = (nthreads + 255) / 256;
        int* blk = talloc<int>(nb, st);
        int64_t* cl = talloc<int64_t>(nb + 1, st);
        int64_t* ce = talloc<int64_t>(nb + 1, st);
        int64_t* ol = talloc<int64_t>(nb + 1, st);
        int64_t* oe = talloc<int64_t>(nb + 1, st);
        uint8_t* outc = talloc<uint8_t>(nthreads, st);
        ExpandArgs a;
        a.outc = outc;
        a.in = cur;
        a.n_in = n_cur;
        a.kid0 = s->lv.kid0 + s->h_off[L];
        a.kid1 = s->lv.kid1 + s->h_off[L];
        a.child = ch;
        a.tv = tv;
        a.blk_counts = blk;
        a.counters = sc;
        a.ledger = sl;
        a.out_expand = nullptr;
        a.out_leaf = nullptr;
        a.blk_off_expand = oe;
        a.blk_off_leaf = ol;
        a.eight = in.sym == 2;
        if (log_ties) {
            if (in.sym) { k_expand<true, false, true><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
            else { k_expand<false, false, true><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
        } else if (in.sym) { k_expand<true, false><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
        else { k_expand<false, false><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
        { k_unpack_counts<<<(unsigned)((nb + 255) / 256), 256, 0, st>>>(blk, nb, cl, ce); note_launch(); }
        HXF_CUDA(cudaMemsetAsync(cl + nb, 0, sizeof(int64_t), st));
        HXF_CUDA(cudaMemsetAsync(ce + nb, 0, sizeof(int64_t), st));
        size_t tb = 0;
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, cl, ol, nb + 1, st));
        void* tbuf = talloc<char>(tb, st);
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, cl, ol, nb + 1, st));
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(tbuf, tb, ce, oe, nb + 1, st));
        int64_t tot[2];
        HXF_CUDA(cudaMemcpyAsync(&tot[0], ol + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaMemcpyAsync(&tot[1], oe + nb, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        const double tr1 = trace ? trav_now_ms() : 0.0;
        HXF_CUDA(cudaStreamSynchronize(st));
        const double tr2 = trace ? trav_now_ms() : 0.0;
        uint64_t* nxt = talloc<uint64_t>(tot[1], st);
        uint64_t* lf = talloc<uint64_t>(tot[0], st);
        if (trace) {
            const double tr3 = trav_now_ms();
            fprintf(stderr, "trav L=%d n=%lld enqueue %.2f sync %.2f alloc %.2f ms\n", L, (long long)n_cur,
                    tr1 - tr0, tr2 - tr1, tr3 - tr2);
        }
        a.out_expand = nxt;
        a.out_leaf = lf;
        if (in.sym) { k_expand<true, true><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
        else { k_expand<false, true><<<(unsigned)nb, 256, 0, st>>>(a); note_launch(); }
        HXF_CUDA(cudaGetLastError());
        for (void* p : {(void*)blk, (void*)cl, (void*)ce, (void*)ol, (void*)oe, tbuf, (void*)cur, (void*)outc})
            hxf_cache_free(p, st);
        if (tot[0]) {
            leaf_parts.push_back(lf);
            leaf_counts.push_back(tot[0]);
        } else {
            hxf_cache_free(lf, st);
        }
        cur = nxt;
        n_cur = tot[1];
        res.frontier_sizes.push_back(n_cur);
    }
    fold_stripes(counters, ledger);
    hxf_cache_free(sc, st);
    hxf_cache_free(sl, st);
    if (discard_top && !cut_reached) {
        // the traversal ended above the cut (a single-leaf system, or a frontier that
        // emptied first): every leaf task belongs to shard 0, none to this shard
        for (uint64_t* p : leaf_parts) hxf_cache_free(p, st);
        leaf_parts.clear();
        leaf_counts.clear();
    }
    if (in.frontier_only) {
        res.frontier = cur;
        res.n_frontier = n_cur;
    } else {
        hxf_cache_free(cur, st);
    }
    // concatenate leaf parts
    int64_t tot = 0;
    for (int64_t c : leaf_counts) tot += c;
    res.leaf = talloc<uint64_t>(tot, st);
    res.n_leaf = tot;
    int64_t off = 0;
    for (size_t k = 0; k < leaf_parts.size(); ++k) {
        HXF_CUDA(cudaMemcpyAsync(res.leaf + off, leaf_parts[k], leaf_counts[k] * sizeof(uint64_t),
                                 cudaMemcpyDeviceToDevice, st));
        off += leaf_counts[k];
        hxf_cache_free(leaf_parts[k], st);
    }
    if (scratch_c) hxf_cache_free(scratch_c, st);
    if (scratch_l) hxf_cache_free(scratch_l, st);
    HXF_CUDA(cudaGetLastError());
    return res;
}
