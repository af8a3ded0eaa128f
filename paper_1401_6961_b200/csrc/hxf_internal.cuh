// Internal types and device helpers shared by the hxf translation units.
#pragma once

#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/hxf.h"

// ---------------------------------------------------------------- errors

void hxf_set_error(const std::string& msg);

struct HxfError {
    int code;
    std::string msg;
};

#define HXF_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            throw HxfError{HXF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)}; \
    } while (0)

// ---------------------------------------------------------------- layout

// One primitive pair of a shell pair (integrals.py:115-154 restated for the
// device): exponent sum p, 1/p, product centre, and
// c = w_a w_b exp(-ab/p |AB|^2) / p * sqrt(2 pi^{5/2}), so the primitive
// (ss|ss) is c_bra c_ket F0(T) / sqrt(p+q).  64-byte aligned record.
// cs = c / sqrt(p): the far-field (ss|ss) closed form c'_b c'_k sqrt(pi)/2 / |P-Q|
// One primitive pair, 64 bytes in two 32-byte halves: {centre, cs} is all the far-field
// (ss|ss) path reads (one 256-bit load), {p, 1/p, c} completes the record (a second one).
struct __align__(32) PrimPair {
    double x, y, z, cs, p, ip, c, pad1;
};

// Partition levels on device (quadtree.py:55-84): spans of every level,
// concatenated; kid indices are level-local indices at the next level; a
// leaf span repeats at deeper levels as its own only child.
struct DevLevels {
    int n_levels;
    int n_leaves;
    const int* off;      // n_levels + 1 (host copy mirrored in HostLevels)
    const int* slo;      // per span (concatenated)
    const int* shi;
    const int* flo;
    const int* fhi;
    const int* kid0;
    const int* kid1;
    const int* leaf_id;  // partition-leaf index or -1
    const int* leaf_span;  // per leaf: span index at the deepest level
};

struct DevBasis {
    int ns;
    int nfn;
    const double3* ctr;
    const int* l;
    const int* poff;
    const int* fn;
    const int* nf;
    const double* exps;
    const double* w;
    const double* sw;
};

// Device state handles (opaque to C callers).
struct hxf_system {
    int device;
    int ns, nfn, n_levels, n_leaves, max_span, max_leaf_shells;
    std::vector<int> h_off, h_slo, h_shi, h_flo, h_fhi, h_kid0, h_kid1, h_leaf_id, h_l, h_poff,
        h_fn, h_nf;
    std::vector<int64_t> node_off;  // per level offset of dense node arrays (n_L^2)
    DevBasis basis;
    DevLevels lv;
    std::vector<void*> allocs;
};

struct hxf_pairs {
    hxf_system* sys;
    int device;
    double tau_ovlp;
    double* norm;      // per level dense; -1 where pruned
    double* rowsum;
    double* colsum;
    double* smax;      // block max |S|
    double* snorm;     // per node: sqrt(diag_norm) (Schwarz task factor), -1 where pruned
    double* srow;      // per node: sqrt(max(rowsum, 0)), sqrt(max(colsum, 0)) (ledger factors)
    double* scol;
    int64_t* leaf_base;  // per leaf pair (nleaf^2): first pair id, -1 if pruned
    int64_t n_pairs;
    int* pi;           // per pair id: shells
    int* pj;
    int64_t* ppoff;    // n_pairs + 1
    double* q;         // per pair id: Q in canonical orientation
    double* sq;        // per pair id: sqrt(Q) (correctly rounded, = math.sqrt)
    uint8_t* meta;     // per pair id: (l_i << 1 | l_j) | (n prim pairs - 1) << 2
    PrimPair* pp;
    int4* info;        // per pair id: {fn offset i, fn offset j, first prim pair, n prim pairs}
    int64_t n_prim_pairs;
    double maxq;
    double amax;       // max over shells s of sum_{pairs (s,t) or (t,s)} n_f(t) sqrt(Q) (K scale bound)
    PrimPair* epp;     // ERI primitive table: each pair's primitives sorted by Schwarz factor, descending
    float4* geo;       // per pair: centroid of the primitive centres, radius (conservative, far-field test)
    float* gip;        // per pair: max 1/p over its primitives (rounded up)
    double* eS;        // per entry of epp: primitive Schwarz factor sqrt(max_comp (ab|ab))
    uint8_t* fcol;     // per pair: 1 = same-centre (ss| pair whose far-field primitive list collapses to the
                       // single point charge stored at epp[n_prim_pairs + pair id] (k_prim_schwarz_sort)
    double smax_prim;  // max eS
    std::vector<hxf_tie_record> ovlp_ties;   // overlap-pruning ties found at build (first 4096)
    int64_t n_ovlp_ties = 0;
    int* ncid;         // per leaf pair node (nleaf^2): compact live-node id, -1 if pruned
    double* nvec;      // per live node: NVEC doubles, row/col max Q and row/col sums of sqrt(Q)
    double* nvec_tri;  // per leaf span (diagonal node, canonical x <= y pairs): the same vectors
    int has_p;
};

// Primitive-quartet neglect in the ERI stage: a primitive pair ab is dropped
// from a build when S_ab * max S_cd * max|P| <= HXF_PRIM_EPS, so every
// dropped primitive quartet's contribution to any K element is <= HXF_PRIM_EPS
// (|(ab|cd)| <= S_ab S_cd, Cauchy-Schwarz on the Coulomb metric).  The
// Schwarz factors Q of the culling tests always use every primitive.
#define HXF_PRIM_EPS 1e-16

// node vectors of a leaf pair node (mu, nu), shells x of mu and y of nu:
//   [NV_FR + x] = max_y Q(x,y)   [NV_FC + y] = max_x Q(x,y)
//   [NV_SR + x] = sum_y sqrtQ    [NV_SC + y] = sum_x sqrtQ
#define NV_MAXS 10
#define NV_FR 0
#define NV_FC NV_MAXS
#define NV_SR (2 * NV_MAXS)
#define NV_SC (3 * NV_MAXS)
//   [NV_GR + x] = sqrt(max_y Q) = max_y sqrtQ   [NV_GC + y] likewise (sqrt is monotone and
//   correctly rounded): the Schwarz-mode cell factors, so the screen takes no square root
#define NV_GR (4 * NV_MAXS)
#define NV_GC (5 * NV_MAXS)
#define NVEC (6 * NV_MAXS)

// Stream-ordered caching allocator for the builds' scratch (api.cu).  Freed blocks
// go to a per-(device, stream, size-bucket) free list instead of back to the CUDA
// pool: cudaMallocAsync stalled for up to ~0.7 s now and then between builds
// (HXF_TRAV_TRACE), so steady-state builds allocate nothing.  A block freed on
// stream s is only reused by later allocations on s (stream order = safety, as
// with cudaFreeAsync).  hxf_cache_free of a pointer it did not allocate falls back
// to cudaFreeAsync.
void* hxf_cache_alloc(size_t bytes, cudaStream_t st);
void hxf_cache_free(void* p, cudaStream_t st);
// free device bytes; hands the cached scratch back first when fewer than `want` are free
size_t hxf_free_memory(size_t want);

struct hxf_density {
    hxf_system* sys;
    int device;
    double* P;         // n x n row-major
    double* norm;      // per level dense; -1 where absent
    double zero_drop;
    double frob;       // root norm
    double maxabs;
    double* pmax;      // n_shells^2: max |P| over each shell-pair function block
};

// ---------------------------------------------------------------- helpers

__host__ __device__ __forceinline__ int64_t node_index(const int64_t* node_off, int level,
                                                       int nspan, int r, int c) {
    return node_off[level] + (int64_t)r * nspan + c;
}

// 256-bit read-only global load (sm_100a LDG.E.256): one instruction, and for the
// scattered per-lane gathers of the ERI kernels one L1 wavefront per lane, per 32 bytes
struct __align__(32) Double4 { double a, b, c, d; };
__device__ __forceinline__ Double4 ldg256(const void* p) {
    Double4 r;
    asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
    return r;
}

__device__ __forceinline__ PrimPair load_pp(const PrimPair* p) {
    const Double4 u = ldg256(p), v = ldg256(reinterpret_cast<const char*>(p) + 32);
    PrimPair r;
    r.x = u.a; r.y = u.b; r.z = u.c; r.cs = u.d;
    r.p = v.a; r.ip = v.b; r.c = v.c; r.pad1 = 0.0;
    return r;
}

// the fields the far-field (ss|ss) path reads: centre and cs
__device__ __forceinline__ PrimPair load_pp_far(const PrimPair* p) {
    const Double4 u = ldg256(p);
    PrimPair r;
    r.x = u.a; r.y = u.b; r.z = u.c; r.cs = u.d;
    r.p = 0.0; r.ip = 0.0; r.c = 0.0; r.pad1 = 0.0;
    return r;
}

// sorted 3-factor product (exchange_naive.py:68-71); no FMA contraction.
__device__ __forceinline__ double sorted_product3(double a, double b, double c) {
    double lo = fmin(a, b), hi = fmax(a, b);
    double mid;
    if (c < lo) { mid = lo; lo = c; }
    else if (c > hi) { mid = hi; hi = c; }
    else mid = c;
    return __dmul_rn(__dmul_rn(lo, mid), hi);
}

// ---------------------------------------------------------------- fsum

// Correctly rounded sum (Shewchuk partials + CPython's final half-way
// correction), so device norms match math.fsum (quadtree.py:20-25) bit for
// bit given identical inputs.  Partials live in local memory.
// Capacity: the partials are non-overlapping doubles; sums of squares that reach down
// into the denormals were seen to need 48-49 of them (a 20 x 20-shell leaf block), so
// the array holds 96, and if it ever fills the running sum is folded into the top
// partial (inexact by an ulp of that partial) instead of being dropped.
#define FSUM_CAP 96
struct FSum {
    double part[FSUM_CAP];
    int n;
    __device__ __forceinline__ FSum() : n(0) {}
    __device__ __forceinline__ void add(double x) {
        int i = 0;
        for (int k = 0; k < n; ++k) {
            double y = part[k];
            if (fabs(x) < fabs(y)) { double t = x; x = y; y = t; }
            double hi = __dadd_rn(x, y);
            double lo = __dsub_rn(y, __dsub_rn(hi, x));
            if (lo != 0.0) part[i++] = lo;
            x = hi;
        }
        if (i < FSUM_CAP) part[i++] = x;
        else part[FSUM_CAP - 1] = __dadd_rn(part[FSUM_CAP - 1], x);
        n = i;
    }
    __device__ __forceinline__ double result() const {
        if (n == 0) return 0.0;
        int k = n - 1;
        double hi = part[k], lo = 0.0;
        while (k > 0) {
            double x = hi;
            --k;
            double y = part[k];
            hi = __dadd_rn(x, y);
            double yr = __dsub_rn(hi, x);
            lo = __dsub_rn(y, yr);
            if (lo != 0.0) break;
        }
        if (k > 0 && ((lo < 0.0 && part[k - 1] < 0.0) || (lo > 0.0 && part[k - 1] > 0.0))) {
            double y = lo * 2.0;
            double x = __dadd_rn(hi, y);
            double yr = __dsub_rn(x, hi);
            if (y == yr) hi = x;
        }
        return hi;
    }
};

// ---------------------------------------------------------------- fixed point
//
// Order-independent accumulation: each value is rounded once to an N-limb
// two's-complement integer at scale 2^S and added with integer atomics, so
// sums are bitwise reproducible regardless of thread scheduling.

template <int N>
__device__ __forceinline__ void fx_from_double(double x, int S, unsigned long long* limb) {
#pragma unroll
    for (int k = 0; k < N; ++k) limb[k] = 0ull;
    if (x == 0.0) return;
    const bool neg = x < 0.0;
    unsigned long long bits = (unsigned long long)__double_as_longlong(fabs(x));
    int ex = (int)((bits >> 52) & 0x7ff);
    unsigned long long mant = bits & ((1ull << 52) - 1);
    if (ex == 0) ex = 1; else mant |= (1ull << 52);
    int s = ex - 1075 + S;  // value = mant * 2^s
    if (s < 0) {
        if (s <= -64) return;
        int sh = -s;
        unsigned long long rem = mant & ((1ull << sh) - 1);
        mant >>= sh;
        unsigned long long half = 1ull << (sh - 1);
        if (rem > half || (rem == half && (mant & 1ull))) mant += 1;
        s = 0;
    }
    int li = s >> 6, off = s & 63;
    if (li < N) limb[li] = mant << off;
    if (off && li + 1 < N) limb[li + 1] = mant >> (64 - off);
    if (neg) {
        unsigned long long carry = 1;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            unsigned long long v = ~limb[k] + carry;
            carry = (carry && v == 0) ? 1ull : 0ull;
            limb[k] = v;
        }
    }
}

template <int N>
__device__ __forceinline__ void fx_atomic_add(unsigned long long* acc, const unsigned long long* v) {
    unsigned long long carry = 0;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        unsigned long long add = v[k] + carry;
        unsigned long long c1 = (add < carry) ? 1ull : 0ull;
        unsigned long long c2 = 0;
        if (add != 0ull) {
            unsigned long long old = atomicAdd(acc + k, add);
            c2 = (old + add < old) ? 1ull : 0ull;
        }
        carry = c1 + c2;
        if (k + 1 < N && carry == 0ull) {
            // remaining limbs of v may still be nonzero (sign extension)
            bool rest = false;
#pragma unroll
            for (int t = k + 1; t < N; ++t) rest |= (v[t] != 0ull);
            if (!rest) break;
        }
    }
}

template <int N>
__host__ __device__ inline double fx_to_double(const unsigned long long* limb, int S) {
    // interpret as signed two's complement
    const bool neg = (long long)limb[N - 1] < 0;
    unsigned long long m[N];
    unsigned long long carry = 1;
    for (int k = 0; k < N; ++k) {
        m[k] = neg ? ~limb[k] + carry : limb[k];
        if (neg) carry = (carry && m[k] == 0) ? 1ull : 0ull;
    }
    double r = 0.0;
    for (int k = N - 1; k >= 0; --k) r = r + ldexp((double)m[k], 64 * k - S);
    return neg ? -r : r;
}

#define LEDGER_LIMBS 4
#define LEDGER_SCALE 160
// K accumulator (per element, 8 B): v = rint(x 2^S) summed with one
// fire-and-forget 64-bit reduction per contribution.  S is chosen per build
// from a rigorous bound B on the sum of |contributions| any element can
// receive (k_scale_bits: B <= 4 A_max^2 max|P|, A(s) = sum over the pairs
// (s,t) of n_f(t) sqrt(Q_st)), so every partial sum stays below 2^62 and
// cannot overflow.  Integer sums are order independent, so K is bitwise
// reproducible; each contribution is rounded once, to 2^-(S+1).
__device__ __forceinline__ void k_fixed_add(unsigned long long* acc, double x, int S) {
    const long long v = __double2ll_rn(ldexp(x, S));  // ldexp by a power of two: exact
    if (v) atomicAdd(acc, (unsigned long long)v);
}

__host__ __device__ inline double k_fixed_value(const unsigned long long* acc, int S) {
    return ldexp((double)(long long)acc[0], -S);
}

// ---------------------------------------------------------------- warp utils

__device__ __forceinline__ void atomic_add_ll(long long* p, long long v) {
    atomicAdd(reinterpret_cast<unsigned long long*>(p), (unsigned long long)v);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ---------------------------------------------------------------- NVTX
// Stage ranges for timeline tools (header-only nvtx3: no library, no cost unless a
// tool is attached): pair tree, density tree, traversal, leaf screen, ERI stage, epilogue.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---------------------------------------------------------------- tie records
// Bounded device log of culling comparisons within 1e-12 (relative) of their
// threshold (hxf_tie_record, include/hxf.h).  Ties are rare: the append is one
// atomic on the cold path of the comparison; count == NULL disables it.
struct TieLog {
    hxf_tie_record* rec;
    unsigned long long* count;
    long long cap;
};

// (never inlined: the hot kernels keep their register budgets; ties are rare)
static __device__ __noinline__ void tie_emit(TieLog tl, int stage, int level, int slot, bool kept, int a,
                                      int b, int c, int d, double bound, double thr) {
    if (!tl.count) return;
    const unsigned long long pos = atomicAdd(tl.count, 1ull);
    if ((long long)pos < tl.cap) {
        hxf_tie_record r;
        r.stage = stage; r.level = level; r.slot = slot; r.decision = kept ? 1 : 0;
        r.id[0] = a; r.id[1] = b; r.id[2] = c; r.id[3] = d;
        r.bound = bound; r.threshold = thr; r.contribution = bound;
        tl.rec[pos] = r;
    }
}

// counter slots in the device counter array
enum {
    C_VISITED = 0, C_CULL_SCREEN, C_CULL_ABSENT, C_LEAF, C_ERIQ, C_CULL_LEAF, C_EXPANDED,
    C_SPAWNED, C_LINK_SCREEN, C_LINK_ABSENT, C_CASE0, C_CASELEAF0 = C_CASE0 + HXF_NCASES,
    C_TIE_TASK = C_CASELEAF0 + HXF_NCASES, C_TIE_LEAF, C_PRIMQ, C_OVERFLOW, C_CLSQ0,
    C_CLSPQ0 = C_CLSQ0 + 16, C_DBG0 = C_CLSPQ0 + 16, C_SCREEN_BYTES = C_DBG0 + 8,
    C_NCOUNTERS = C_SCREEN_BYTES + 1
};

// Device-side bounds checks (build with -DHXF_DEBUG_BOUNDS; compute-sanitizer is not
// available on the GPU pool): a failed check counts in counters[C_OVERFLOW] and the
// access is skipped; the build then fails with HXF_ELOGIC.  Off: no code.
#ifdef HXF_DEBUG_BOUNDS
#define HXF_BCHECK(cond, counters) \
    ((cond) ? true : (atomicAdd(reinterpret_cast<unsigned long long*>(&(counters)[C_OVERFLOW]), 1ull), false))
#else
#define HXF_BCHECK(cond, counters) true
#endif

// kernels launched by the library (evidence that the device path ran)
void note_launch(int n = 1);

// ---------------------------------------------------------------- launchers
// (defined in the .cu files)

// pageable host <-> device transfers of the boundary's n^2 arrays (xfer.cu): return when done
void xfer_to_device(void* dst_dev, const void* src_host, size_t bytes, cudaStream_t st);
void xfer_to_host(void* dst_host, const void* src_dev, size_t bytes, cudaStream_t st);

void launch_boys_init();
void trees_build_pairs(hxf_pairs* pr, cudaStream_t st, const double* s_user = nullptr);
void trees_build_density(hxf_density* d, const double* P, int on_device, cudaStream_t st);

struct ExchangeCtx;
int direct_run(hxf_pairs* pairs, hxf_density* dens, const hxf_exchange_opts* o, double* K_out,
               hxf_counters* out, cudaStream_t st);
int exchange_run(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, const hxf_exchange_opts* o,
                 double* K_out, hxf_counters* c, cudaStream_t st);
int symmetrize_device(double* K, int n, double tol, cudaStream_t st);
double fp64_peak(cudaStream_t st);
int frontier_run(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, double tau, int mode, int sym,
                 int level, int64_t* n_tasks, double* cost, int64_t cap, cudaStream_t st);
