/*
 * hxf.h -- C ABI of libhxf.so, the B200 (sm_100a) hierarchical exchange build.
 *
 * Drop-in boundary for the reference's hot path (paths relative to
 * /root/reference/pkg/src/hexfock).  Each entry point replaces one reference
 * interface; the Python mirror (paper_1401_6961_b200/quadtree.py,
 * exchange.py) binds them with ctypes and keeps the reference signatures.
 *
 *   hxf_system_create   <- build_partition (quadtree.py:90-113) output + the
 *                          BasisSystem / GaussianShell inputs (basis.py:62-101)
 *   hxf_pairs_build     <- build_pair_tree            (quadtree.py:284-337)
 *   hxf_density_build   <- build_matrix_tree          (quadtree.py:198-235)
 *   hxf_exchange        <- build_exchange_naive       (exchange_naive.py:200-240)
 *                          build_exchange_symmetric   (exchange_symmetry.py:364-409)
 *   hxf_*_download      <- node attribute reads of ShellPairNode /
 *                          MatrixQuadtree (quadtree.py:116-142, 238-269)
 *
 * Plain pointers and sizes only; no C++ or torch types.  Every function
 * returns HXF_OK (0) or an error code; hxf_last_error() gives the message of
 * the last failure on the calling thread.  Calls on one object are not
 * thread-safe; use one object per thread.  `stream` is a cudaStream_t (NULL =
 * legacy default stream).
 */
#ifndef HXF_H
#define HXF_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HXF_OK 0
#define HXF_EINVAL 1 /* InvalidArgumentError (basis.py:35-36)           */
#define HXF_ELOGIC 2 /* LogicError (exchange_naive.py:24-25)            */
#define HXF_ECUDA 3  /* CUDA runtime failure / no device                */
#define HXF_ENOMEM 4 /* device allocation failed                        */

#define HXF_MODE_SCHWARZ 0 /* exchange_naive.py:83-85: sqrt of diag norms */
#define HXF_MODE_LITERAL 1 /* exchange_naive.py:86: norms as-is           */

#define HXF_NAIVE 0     /* exchange_naive.py, ordered shell pairs      */
#define HXF_FOURFOLD 1  /* exchange_symmetry.py, canonical pairs       */
#define HXF_EIGHTFOLD 2 /* (new) fourfold folded bra<->ket: canonical pairs, bra pair <= ket pair;
                           K = A + A^T (SURVEY.md 8(a) S8 optional mode)                        */

#define HXF_NCASES 9 /* CASE_LABELS, exchange_symmetry.py:43 */

typedef struct hxf_system hxf_system;   /* basis + partition, device resident */
typedef struct hxf_pairs hxf_pairs;     /* shell-pair quadtree               */
typedef struct hxf_density hxf_density; /* density quadtree + dense P        */

/* TraversalCounters (exchange_naive.py:28-65) + SymmetryCounters extras
 * (exchange_symmetry.py:72-132) + tie counts. */
typedef struct hxf_counters {
    int64_t tasks_visited;
    int64_t tasks_culled_screening;
    int64_t tasks_culled_absent;
    int64_t leaf_contractions;
    int64_t eri_shell_quartets;
    int64_t quartets_culled_leaf;
    int64_t tasks_expanded;
    int64_t children_spawned;
    int64_t links_culled_screening;
    int64_t links_culled_absent;
    int64_t case_tasks[HXF_NCASES];
    int64_t case_leaf_tasks[HXF_NCASES];
    int64_t ties_task;   /* task-level bounds within 1e-12 rel of tau   */
    int64_t ties_leaf;   /* quartet-level bounds within 1e-12 rel of tau */
    int64_t prim_quartets; /* primitive quartets evaluated (work metric) */
    int64_t class_quartets[16];      /* evaluated shell quartets per (li,lj,lk,ll) class */
    int64_t class_prim_quartets[16]; /* primitive quartets per class                    */
    double culled_bound_ledger;
    /* leaf screen, algorithmic bytes: per leaf task 8 (m_bra + m_ket)
       of Q plus 8 n_row n_col of the |P| block per live slot; filled only when
       hxf_exchange_opts.count_screen_bytes is set */
    int64_t screen_bytes;
} hxf_counters;

/* One culling comparison whose bound lies within 1e-12 (relative) of its threshold
 * (BASELINE north star: "such ties must be logged").  The
 * device takes the decision the reference's rule gives for its own bound; a tie is
 * where a bound computed a few ulps differently could decide the other way. */
#define HXF_TIE_TASK 0      /* traversal: (lo*mid)*hi <= tau (exchange_naive.py:68-88)   */
#define HXF_TIE_LEAF 1      /* leaf quartet: (f(Q_ij)|P|)f(Q_kl) > tau (:156-182)        */
#define HXF_TIE_OVERLAP 2   /* pair-tree pruning: block max |S| < tau_ovlp (quadtree.py:296-299) */
typedef struct hxf_tie_record {
    int32_t stage;         /* HXF_TIE_*                                               */
    int32_t level;         /* task / overlap: partition level of the node(s); leaf: -1 */
    int32_t slot;          /* fourfold slot g (0: naive, overlap)                      */
    int32_t decision;      /* 1: kept / expanded / live, 0: culled / pruned            */
    int32_t id[4];         /* task: level-local span indices mu,nu,lam,sig; leaf: shell
                              ids i,j,k,l; overlap: level-local span indices r,c,-1,-1 */
    double bound;
    double threshold;
    double contribution;   /* task / leaf: upper bound on the K change a flipped decision
                              could cause (= bound); overlap: the block max |S|        */
} hxf_tie_record;

/* Exchange options.  The shard fields select a subset of the product-tree
 * tasks at level `shard_level` (tasks [shard_begin, shard_end) of that
 * level's frontier, in frontier order, every shard_stride-th one when
 * shard_stride > 1) for multi-GPU runs; shard_level < 0 runs the whole tree. */
typedef struct hxf_exchange_opts {
    double tau_2e;
    int mode;          /* HXF_MODE_*   */
    int symmetry;      /* HXF_NAIVE / HXF_FOURFOLD / HXF_EIGHTFOLD */
    int evaluate;      /* 0: counters only, K = 0 (exchange_naive.py:183) */
    int K_on_device;   /* K_out is a device pointer                  */
    int symmetrize;    /* fourfold: apply symmetrize_final (:197-209) */
    int shard_level;
    int64_t shard_begin;
    int64_t shard_end;
    int32_t* quartet_log;   /* NULL or 4*capacity int32 (host) */
    int64_t log_capacity;
    int64_t* log_count;     /* out: quartets logged (may exceed capacity) */
    /* Order-independent digest of the evaluated quartet set (SURVEY.md 8(c)
       item 2: full-size parity without a materialised log).  NULL, or host
       uint64[3] = {count, sum h(q), sum h(h(q))} mod 2^64 over the evaluated
       tuples q = (i,j,k,l) (the quartet_log tuples) with i % digest_mod ==
       digest_rem; h = SplitMix64 finaliser of ((i*ns + j)*ns + k)*ns + l.
       Filled only when evaluate != 0. */
    uint64_t* digest;
    int digest_mod;    /* <= 1: every quartet */
    int digest_rem;
    /* K_fixed != 0 (requires K_on_device): K_out receives the signed 64-bit
       fixed-point accumulator (int64 n x n, value = v * 2^-S) instead of FP64 K,
       and *K_scale = S.  S depends only on (bra, ket, P), so shards of one build
       share it and their partials sum exactly (integer all-reduce);
       hxf_fixed_to_double converts.  symmetrize is ignored. */
    int K_fixed;
    int* K_scale;
    /* <= 1: contiguous shard range; s > 1: tasks shard_begin, shard_begin + s,
       ... below shard_end (cyclic assignment: rank r of N takes begin r, stride N) */
    int64_t shard_stride;
    /* NULL, or host uint8[shard_end]: shard = the frontier tasks t < shard_end
       with shard_mask[t] != 0 (any assignment, e.g. cost-balanced); the range /
       stride fields are then ignored except that work above the cut is counted
       only when shard_begin == 0 */
    const uint8_t* shard_mask;
    /* Start node of the traversal: the diagonal node (root_index, root_index) of
       partition level root_level (0, 0 = the tree root).  The reference's drivers
       accept any node with bra.row is bra.col is ket.row ... is P.col
       (exchange_naive.py:105-108 _check_same_partition); K_out is then the
       n_S x n_S block of that span's functions (n_S = its function count, local
       indices fn - fn_lo).  K_fixed requires the tree root. */
    int root_level;
    int root_index;
    /* Tie records of this build (task and leaf stages): NULL, or a host array of
       tie_capacity records; *tie_count (may be NULL) receives the number of ties
       found, which may exceed the capacity.  The counters' ties_task / ties_leaf
       are filled either way.  Overlap-stage ties belong to the pair tree:
       hxf_pairs_ties. */
    hxf_tie_record* tie_log;
    int64_t tie_capacity;
    int64_t* tie_count;
    /* != 0: also fill counters.screen_bytes (one extra pass over the leaf task list;
       a measurement aid for the leaf-screen roofline, off in normal builds) */
    int count_screen_bytes;
} hxf_exchange_opts;

const char* hxf_last_error(void);
int hxf_version(void);

int hxf_system_create(int device, int n_shells, const double* centers /* ns*3 Bohr */,
                      const int* l /* 0|1 */, const int* prim_off /* ns+1 */,
                      const double* exponents, const double* weights,
                      const double* s_weights /* s-normalised weights for overlap pruning */,
                      int n_levels, const int* level_off /* n_levels+1 */,
                      const int* span_shell_lo, const int* span_shell_hi,
                      const int* span_fn_lo, const int* span_fn_hi,
                      const int* span_kid0, const int* span_kid1 /* level-local, -1 none */,
                      hxf_system** out);
void hxf_system_destroy(hxf_system* sys);
int hxf_system_info(const hxf_system* sys, int64_t* n_functions, int64_t* n_leaves);

int hxf_pairs_build(hxf_system* sys, double tau_ovlp, void* stream, hxf_pairs** out);
/* build_pair_tree(..., overlap_matrix=S) (quadtree.py:284-293): pruning from the
 * caller's |S| (n_shells x n_shells row-major, float64, absolute values; host or
 * device per on_device) instead of the computed overlaps: a node is pruned iff
 * max |S| over its (row span, column span) block < tau_ovlp.  S is not assumed
 * symmetric.  Q, the primitive tables and the ERIs are unchanged. */
int hxf_pairs_build_ovlp(hxf_system* sys, double tau_ovlp, const double* s_abs, int on_device,
                         void* stream, hxf_pairs** out);
void hxf_pairs_destroy(hxf_pairs* pairs);
/* node arrays of one level (n_spans(level)^2 entries, row-major (r, c)):
 * diag_norm, rowsum_max, colsum_max, pruned flag (1 = pruned). */
int hxf_pairs_download(const hxf_pairs* pairs, int level, double* diag_norm, double* rowsum_max,
                       double* colsum_max, uint8_t* pruned);
/* Q = (ij|ij) (max over function pairs for p), n_shells^2 row-major; entries
 * outside live leaf nodes are set to -1. */
int hxf_pairs_download_q(const hxf_pairs* pairs, double* q);
/* |S_ij| (s-proxy contracted overlap), n_shells^2 row-major. */
int hxf_pairs_overlap(const hxf_pairs* pairs, double* s_abs);

int hxf_density_build(hxf_system* sys, const double* P, int P_on_device, double zero_drop,
                      void* stream, hxf_density** out);
void hxf_density_destroy(hxf_density* dens);
/* node norms of one level, -1 where the node is absent. */
int hxf_density_download(const hxf_density* dens, int level, double* norm);
/* max |P| over each shell block (the per-quartet bound's density factor for
 * p shells), n_shells^2 row-major. */
int hxf_density_download_pmax(const hxf_density* dens, double* pmax);

int hxf_exchange(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, const hxf_exchange_opts* opts,
                 double* K_out, hxf_counters* counters, void* stream);
/* K[t] = Kfx[t] * 2^-S for t < n2 (device arrays; may alias: in place). */
int hxf_fixed_to_double(const int64_t* Kfx, int64_t n2, int S, double* K, void* stream);

/* Direct-SCF twin (dense_exchange_screened, oracle.py:69-108; SURVEY.md 8(f)
 * f1): every ordered shell quartet of live pairs with
 * (f(Q_ij) |P|_jk) f(Q_kl) > tau_2e, enumerated without the hierarchy and
 * evaluated by the same ERI stage into the same fixed-point K, so its K equals
 * the naive hierarchical K bit for bit when the evaluated sets agree.  Uses
 * opts->tau_2e, mode, evaluate, K_on_device, digest; digest_mod/digest_rem
 * restrict the EVALUATED quartets to first shells i % mod == rem (sampled K
 * rows).  Counters: eri_shell_quartets, prim_quartets and the class arrays. */
int hxf_exchange_direct(hxf_pairs* pairs, hxf_density* P, const hxf_exchange_opts* opts,
                        double* K_out, hxf_counters* counters, void* stream);

/* Frontier size of the product tree at `level` (for multi-GPU shard
 * planning); also returns per-task cost estimates (descendant leaf count
 * proxy) when `cost` is non-NULL (host buffer of that size). */
int hxf_frontier(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, double tau_2e, int mode,
                 int symmetry, int level, int64_t* n_tasks, double* cost, int64_t cost_capacity,
                 void* stream);

/* Symmetrise a device K in place: LogicError if max|K - K^T| > tol, else
 * K = (K + K^T)/2 (symmetrize_final, exchange_symmetry.py:197-209); used after
 * the multi-GPU reduction of partial K. */
int hxf_symmetrize(double* K_dev, int n, double tol, void* stream);

/* FP64 FMA throughput of the current device (TFLOP/s, FMA = 2 flops),
 * measured with a dependent-chain-free DFMA kernel over all SMs. */
int hxf_fp64_peak(double* tflops, void* stream);

/* Device Hilbert reordering of shells (replaces the host
 * pre-pass hilbert_order / hilbert_index_3d, reference basis.py:275-331).
 * centers: n x 3 float64 row-major (Bohr); bits = bits_per_axis in [1, 20]
 * (HXF_EINVAL otherwise, same message as basis.py:311-312).  perm[k] = index of
 * the shell placed k-th (numpy argsort(keys, kind="stable")); keys (may be
 * NULL) receives the keys in sorted order.  on_device != 0: all three are
 * device pointers and the call is stream-ordered on `stream`; 0: host pointers,
 * copied in and out, returns after the copy back.  Bitwise the host result. */
int hxf_hilbert_order(const double* centers, int64_t n, int bits, int on_device, int64_t* perm,
                      uint64_t* keys, void* stream);

/* Device partition build (replaces build_partition, reference
 * quadtree.py:90-113): recursive bisection of the shells at the boundary nearest
 * the function midpoint, ties left, until a span holds <= leaf_size functions.
 * shell_nfunc: host int32 function count per shell.  Output (host buffers): the
 * spans level by level as in Partition.levels (a leaf repeats at deeper levels):
 * level k is span_lo/span_hi[level_off[k] .. level_off[k+1]).  *n_spans and
 * *n_levels receive the sizes; if span_capacity or level_capacity (>= levels+1
 * entries of level_off) is too small nothing is written but the two sizes and
 * HXF_EINVAL is returned.  leaf_size below the largest shell: HXF_EINVAL with
 * the reference's message.  Identical spans to the host rules. */
int hxf_partition_build(const int32_t* shell_nfunc, int64_t n_shells, int leaf_size,
                        int32_t* span_lo, int32_t* span_hi, int64_t span_capacity,
                        int64_t* level_off, int level_capacity, int64_t* n_spans, int* n_levels,
                        void* stream);

/* Block-sparse reduction of shard K accumulators (the
 * multi-GPU all-reduce of exchange_sharded, csrc/reduce.cu).  All arrays are
 * device arrays; K is the n x n int64 fixed-point accumulator, tiles are bs x bs
 * (nb = ceil(n / bs), nb * nb tiles, row-major, edge tiles zero-padded).
 * hxf_block_mask: mask[t] = 1 if tile t holds a nonzero.
 * hxf_block_slots: slot[0..nt] = exclusive prefix sum of mask (nt + 1 entries);
 *   *n_blocks (host) = number of flagged tiles (synchronises the stream).
 * hxf_block_pack / hxf_block_unpack: copy flagged tiles K <-> buf (n_blocks * bs^2
 *   int64); unpack writes only flagged tiles.
 * Any 8-byte aligned K / buf is accepted (16-byte accesses are used only when
 * n and bs are even and both pointers are 16-byte aligned); more than
 * 2^31 - 1 tiles is HXF_EINVAL. */
int hxf_block_mask(const int64_t* K, int n, int bs, uint8_t* mask, void* stream);
int hxf_block_slots(const uint8_t* mask, int64_t n_tiles, int64_t* slot, int64_t* n_blocks, void* stream);
int hxf_block_pack(const int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, int64_t* buf,
                   void* stream);
int hxf_block_unpack(int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, const int64_t* buf,
                     void* stream);

/* K quadtree leaves and the row-owning reduce-scatter (second part; the
 * reference treats K as a quadtree over the same index bisection as P, PAPER.md:174-198;
 * csrc/reduce.cu).  Leaf tile (r, c) = rows [flo[r], fhi[r]) x cols [flo[c], fhi[c]) of the
 * partition's leaf spans (device int32 arrays of nleaf entries, the function ranges of
 * quadtree.py:28-60's leaf Spans in order).
 * hxf_span_mask: mask[r * nleaf + c] = 1 if leaf tile (r, c) of the n x n int64 K holds a nonzero.
 * hxf_span_pack / hxf_span_unpack: move the flagged tiles of row spans [r0, r1) between K and
 *   buf; tile (r, c) lives at buf + off[r * nleaf + c] - off_base, row-major inside (off: the
 *   caller's exclusive scan of mask * tile size, in elements).  K addresses matrix row i at
 *   K + (i - row_base) * n, so K may be a row block of the matrix.
 * hxf_fixed_fold: K <- K + K^T in place (exact integer adds). */
int hxf_span_mask(const int64_t* K, int n, const int32_t* flo, const int32_t* fhi, int nleaf, uint8_t* mask,
                  void* stream);
int hxf_span_pack(const int64_t* K, int n, int row_base, const int32_t* flo, const int32_t* fhi, int nleaf,
                  int r0, int r1, const uint8_t* mask, const int64_t* off, int64_t off_base, int64_t* buf,
                  void* stream);
int hxf_span_unpack(int64_t* K, int n, int row_base, const int32_t* flo, const int32_t* fhi, int nleaf,
                    int r0, int r1, const uint8_t* mask, const int64_t* off, int64_t off_base, const int64_t* buf,
                    void* stream);
int hxf_fixed_fold(int64_t* K, int n, void* stream);

/* Overlap-pruning ties of a pair tree: nodes whose block max |S| lies within 1e-12
 * (relative) of tau_ovlp, found when the tree was built.  Copies up to `capacity`
 * records (out may be NULL) and sets *count to the number found. */
int hxf_pairs_ties(const hxf_pairs* p, hxf_tie_record* out, int64_t capacity, int64_t* count);

/* Number of kernels libhxf has launched in this process (work evidence). */
int hxf_launch_count(int64_t* n);

/* Build scratch is cached across builds (per device, stream and size bucket) so
 * steady-state builds allocate nothing.  This synchronises the current device
 * and returns every cached block to the CUDA pool; *bytes (may be NULL)
 * receives the bytes released. */
int hxf_scratch_release(int64_t* bytes);

/* Device timing of the last hxf_exchange on this thread (ms per stage):
 * [0] traversal, [1] leaf screen, [2] ERI stage (far-field classification + sort +
 * ERI kernels), [3] epilogue, [4] total, [5] ERI + contraction kernels only,
 * [6] far-field classification + survivor sort + key bounds. */
int hxf_last_timings(double* ms, int n);

#ifdef __cplusplus
}
#endif
#endif /* HXF_H */
