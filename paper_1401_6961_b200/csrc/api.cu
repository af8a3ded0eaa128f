// C ABI of libhxf.so (include/hxf.h): argument validation, device state
// ownership, error codes.  All compute lives in trees.cu / traverse.cu / leaf.cu.

#include <atomic>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <unordered_map>
#include <vector>

#include "hxf_internal.cuh"

static thread_local std::string g_err;

void hxf_set_error(const std::string& msg) { g_err = msg; }

static std::atomic<int64_t> g_launches{0};
void note_launch(int n) { g_launches += n; }

int hxf_last_timings_impl(double* ms, int n);
int fixed_to_double_impl(const int64_t* Kfx, int64_t n2, int S, double* K, cudaStream_t st);
void block_mask_device(const int64_t* K, int n, int bs, uint8_t* mask, cudaStream_t st);
void span_mask_device(const int64_t* K, int n, const int* flo, const int* fhi, int nleaf, uint8_t* mask,
                      cudaStream_t st);
void span_move_device(int64_t* K, int n, int row_base, const int* flo, const int* fhi, int nleaf, int r0, int r1,
                      const uint8_t* mask, const int64_t* off, int64_t off_base, int64_t* buf, bool pack,
                      cudaStream_t st);
void fold_fixed_device(int64_t* K, int n, cudaStream_t st);
int64_t block_slots_device(const uint8_t* mask, int64_t nt, int64_t* slot, cudaStream_t st);
void block_move_device(int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, int64_t* buf,
                       bool pack, cudaStream_t st);
void partition_build_device(const int32_t* sizes, int n, int leaf, std::vector<int64_t>& level_off,
                            std::vector<int32_t>& span_lo, std::vector<int32_t>& span_hi,
                            cudaStream_t st);
void hilbert_order_device(const double* centers, int64_t n, int bits, int64_t* perm,
                          uint64_t* keys_out, cudaStream_t st);

#define HXF_TRY(...)                                         \
    try {                                                    \
        __VA_ARGS__;                                         \
        return HXF_OK;                                       \
    } catch (const HxfError& e) {                            \
        g_err = e.msg;                                       \
        return e.code;                                       \
    } catch (const std::exception& e) {                      \
        g_err = e.what();                                    \
        return HXF_ECUDA;                                    \
    }

namespace {

template <typename T>
T* upload(const T* h, size_t n, std::vector<void*>& owned) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess)
        throw HxfError{HXF_ENOMEM, "device allocation failed"};
    owned.push_back(p);
    if (n) HXF_CUDA(cudaMemcpy(p, h, n * sizeof(T), cudaMemcpyHostToDevice));
    return (T*)p;
}

void set_device(int dev) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw HxfError{HXF_ECUDA, "no CUDA device available (libhxf has no CPU fallback)"};
    if (dev < 0 || dev >= n) throw HxfError{HXF_EINVAL, "device index out of range"};
    HXF_CUDA(cudaSetDevice(dev));
    // keep stream-ordered allocations cached across builds (no release at sync)
    static thread_local int configured = -1;
    if (configured != dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t thr = UINT64_MAX;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
        configured = dev;
    }
}

struct ScratchCache {
    std::mutex mu;
    std::map<std::tuple<int, cudaStream_t, size_t>, std::vector<void*>> free_lists;
    std::unordered_map<void*, std::pair<cudaStream_t, size_t>> live;  // ptr -> (unused, bucket)
    std::unordered_map<void*, int> dev_of;
};

ScratchCache& scratch_cache() {
    static ScratchCache* c = new ScratchCache();  // never destroyed (outlives CUDA teardown)
    return *c;
}

// size buckets 2^k and 3 * 2^(k-1): at most a third of a block is slack
size_t bucket_of(size_t b) {
    if (b <= 256) return 256;
    size_t p = 256;
    while (p < b) p <<= 1;
    return b <= p / 4 * 3 ? p / 4 * 3 : p;
}

}  // namespace

void* hxf_cache_alloc(size_t bytes, cudaStream_t st) {
    int dev = 0;
    cudaGetDevice(&dev);
    const size_t bk = bucket_of(std::max<size_t>(bytes, 1));
    ScratchCache& c = scratch_cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto it = c.free_lists.find(std::make_tuple(dev, st, bk));
        if (it != c.free_lists.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            c.live[p] = {st, bk};
            return p;
        }
    }
    void* p = nullptr;
    cudaError_t e = cudaMallocAsync(&p, bk, st);
    if (e != cudaSuccess) {  // out of memory: hand every cached block of this device back, retry
        (void)cudaGetLastError();
        {
            std::lock_guard<std::mutex> g(c.mu);
            for (auto& kv : c.free_lists) {
                if (std::get<0>(kv.first) != dev) continue;
                for (void* q : kv.second) {
                    cudaFreeAsync(q, std::get<1>(kv.first));
                    c.dev_of.erase(q);
                }
                kv.second.clear();
            }
        }
        cudaDeviceSynchronize();
        e = cudaMallocAsync(&p, bk, st);
        if (e != cudaSuccess)
            throw HxfError{HXF_ENOMEM, std::string("device allocation failed: ") + cudaGetErrorString(e)};
    }
    std::lock_guard<std::mutex> g(c.mu);
    c.live[p] = {st, bk};
    c.dev_of[p] = dev;
    return p;
}

// Free device memory for sizing a build's survivor buffers: when less than `want` bytes are
// free, the cached scratch blocks of earlier builds (other sizes, other drivers) are handed
// back first -- a cache that starves the next build's chunk capacity defeats its purpose.
size_t hxf_free_memory(size_t want) {
    size_t freeb = 0, totb = 0;
    cudaMemGetInfo(&freeb, &totb);
    if (freeb >= want) return freeb;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceSynchronize();
    ScratchCache& c = scratch_cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        for (auto& kv : c.free_lists) {
            if (std::get<0>(kv.first) != dev) continue;
            for (void* q : kv.second) {
                cudaFree(q);
                c.dev_of.erase(q);
            }
            kv.second.clear();
        }
    }
    cudaMemGetInfo(&freeb, &totb);
    return freeb;
}


void hxf_cache_free(void* p, cudaStream_t st) {
    if (!p) return;
    ScratchCache& c = scratch_cache();
    {
        std::lock_guard<std::mutex> g(c.mu);
        auto it = c.live.find(p);
        if (it != c.live.end()) {
            const size_t bk = it->second.second;
            c.live.erase(it);
            c.free_lists[std::make_tuple(c.dev_of[p], st, bk)].push_back(p);
            return;
        }
    }
    cudaFreeAsync(p, st);
}

extern "C" {

const char* hxf_last_error(void) { return g_err.c_str(); }

int hxf_version(void) { return 1; }

int hxf_system_create(int device, int ns, const double* centers, const int* l, const int* prim_off,
                      const double* exps, const double* weights, const double* s_weights,
                      int n_levels, const int* level_off, const int* slo, const int* shi,
                      const int* flo, const int* fhi, const int* kid0, const int* kid1,
                      hxf_system** out) {
    HXF_TRY({
        if (!out) throw HxfError{HXF_EINVAL, "out is NULL"};
        *out = nullptr;
        if (ns < 1 || n_levels < 1) throw HxfError{HXF_EINVAL, "empty basis or partition"};
        set_device(device);
        hxf_system* s = new hxf_system();
        s->device = device;
        s->ns = ns;
        s->n_levels = n_levels;
        s->h_off.assign(level_off, level_off + n_levels + 1);
        const int nsp = s->h_off[n_levels];
        s->h_slo.assign(slo, slo + nsp);
        s->h_shi.assign(shi, shi + nsp);
        s->h_flo.assign(flo, flo + nsp);
        s->h_fhi.assign(fhi, fhi + nsp);
        s->h_kid0.assign(kid0, kid0 + nsp);
        s->h_kid1.assign(kid1, kid1 + nsp);
        s->h_l.assign(l, l + ns);
        s->h_poff.assign(prim_off, prim_off + ns + 1);
        s->h_fn.resize(ns);
        s->h_nf.resize(ns);
        int off = 0;
        for (int i = 0; i < ns; ++i) {
            if (l[i] != 0 && l[i] != 1) throw HxfError{HXF_EINVAL, "only s and p shells are supported"};
            const int np = prim_off[i + 1] - prim_off[i];
            if (np < 1 || np > 3) throw HxfError{HXF_EINVAL, "shells must have 1..3 primitives"};
            s->h_fn[i] = off;
            s->h_nf[i] = l[i] ? 3 : 1;
            off += s->h_nf[i];
        }
        s->nfn = off;
        // leaf ids: a span is a partition leaf iff it repeats as its own only child
        // (or sits on the deepest level); ids follow deepest-level order
        const int D = n_levels - 1;
        s->h_leaf_id.assign(nsp, -1);
        s->max_span = 0;
        for (int L = 0; L < n_levels; ++L) {
            const int n = s->h_off[L + 1] - s->h_off[L];
            s->max_span = std::max(s->max_span, n);
            if (n > 32767) throw HxfError{HXF_EINVAL, "more than 32767 spans on one partition level"};
        }
        s->n_leaves = s->h_off[D + 1] - s->h_off[D];
        s->max_leaf_shells = 0;
        for (int k = s->h_off[D]; k < s->h_off[D + 1]; ++k) {
            s->h_leaf_id[k] = k - s->h_off[D];
            s->max_leaf_shells = std::max(s->max_leaf_shells, s->h_shi[k] - s->h_slo[k]);
        }
        for (int L = D - 1; L >= 0; --L)
            for (int k = s->h_off[L]; k < s->h_off[L + 1]; ++k)
                if (s->h_kid1[k] < 0) s->h_leaf_id[k] = s->h_leaf_id[s->h_off[L + 1] + s->h_kid0[k]];
        if (s->h_fhi[s->h_off[0]] != s->nfn) throw HxfError{HXF_EINVAL, "partition does not cover the basis"};
        s->node_off.resize(n_levels + 1);
        s->node_off[0] = 0;
        for (int L = 0; L < n_levels; ++L) {
            const int64_t n = s->h_off[L + 1] - s->h_off[L];
            s->node_off[L + 1] = s->node_off[L] + n * n;
        }
        // basis
        std::vector<double3> ctr(ns);
        for (int i = 0; i < ns; ++i) ctr[i] = make_double3(centers[3 * i], centers[3 * i + 1], centers[3 * i + 2]);
        const int npr = prim_off[ns];
        s->basis.ns = ns;
        s->basis.nfn = s->nfn;
        s->basis.ctr = upload(ctr.data(), ns, s->allocs);
        s->basis.l = upload(l, ns, s->allocs);
        s->basis.poff = upload(prim_off, ns + 1, s->allocs);
        s->basis.fn = upload(s->h_fn.data(), ns, s->allocs);
        s->basis.nf = upload(s->h_nf.data(), ns, s->allocs);
        s->basis.exps = upload(exps, npr, s->allocs);
        s->basis.w = upload(weights, npr, s->allocs);
        s->basis.sw = upload(s_weights, npr, s->allocs);
        s->lv.n_levels = n_levels;
        s->lv.n_leaves = s->n_leaves;
        s->lv.off = upload(s->h_off.data(), s->h_off.size(), s->allocs);
        s->lv.slo = upload(slo, nsp, s->allocs);
        s->lv.shi = upload(shi, nsp, s->allocs);
        s->lv.flo = upload(flo, nsp, s->allocs);
        s->lv.fhi = upload(fhi, nsp, s->allocs);
        s->lv.kid0 = upload(kid0, nsp, s->allocs);
        s->lv.kid1 = upload(kid1, nsp, s->allocs);
        s->lv.leaf_id = upload(s->h_leaf_id.data(), nsp, s->allocs);
        s->lv.leaf_span = nullptr;
        *out = s;
    })
}

void hxf_system_destroy(hxf_system* s) {
    if (!s) return;
    cudaSetDevice(s->device);
    for (void* p : s->allocs) cudaFree(p);
    delete s;
}

int hxf_system_info(const hxf_system* s, int64_t* n_functions, int64_t* n_leaves) {
    HXF_TRY({
        if (!s) throw HxfError{HXF_EINVAL, "NULL system"};
        if (n_functions) *n_functions = s->nfn;
        if (n_leaves) *n_leaves = s->n_leaves;
    })
}

static void pairs_build(hxf_system* s, double tau_ovlp, const double* s_abs, int on_device, void* stream,
                        hxf_pairs** out) {
    if (!s || !out) throw HxfError{HXF_EINVAL, "NULL argument"};
    if (!(tau_ovlp >= 0.0)) throw HxfError{HXF_EINVAL, "tau_ovlp must be non-negative"};
    set_device(s->device);
    const cudaStream_t st = (cudaStream_t)stream;
    hxf_pairs* p = new hxf_pairs();
    memset(p, 0, sizeof(*p));
    p->sys = s;
    p->device = s->device;
    p->tau_ovlp = tau_ovlp;
    double* s_dev = nullptr;
    try {
        if (s_abs && !on_device) {  // the caller's |S| (host): staged for the leaf block maxima
            const size_t bytes = (size_t)s->ns * s->ns * sizeof(double);
            HXF_CUDA(cudaMalloc(&s_dev, bytes));
            HXF_CUDA(cudaMemcpyAsync(s_dev, s_abs, bytes, cudaMemcpyHostToDevice, st));
        }
        trees_build_pairs(p, st, s_abs ? (on_device ? s_abs : s_dev) : nullptr);
        if (s_dev) {
            HXF_CUDA(cudaStreamSynchronize(st));
            cudaFree(s_dev);
        }
    } catch (...) {
        if (s_dev) cudaFree(s_dev);
        hxf_pairs_destroy(p);
        throw;
    }
    *out = p;
}

int hxf_pairs_build(hxf_system* s, double tau_ovlp, void* stream, hxf_pairs** out) {
    HXF_TRY({ pairs_build(s, tau_ovlp, nullptr, 0, stream, out); })
}

int hxf_pairs_build_ovlp(hxf_system* s, double tau_ovlp, const double* s_abs, int on_device, void* stream,
                         hxf_pairs** out) {
    HXF_TRY({
        if (!s_abs) throw HxfError{HXF_EINVAL, "NULL overlap matrix"};
        pairs_build(s, tau_ovlp, s_abs, on_device, stream, out);
    })
}

void hxf_pairs_destroy(hxf_pairs* p) {
    if (!p) return;
    cudaSetDevice(p->device);
    void* ptrs[] = {p->norm, p->rowsum, p->colsum, p->smax, p->leaf_base, p->pi,
                    p->pj,   p->ppoff,  p->q,      p->pp,       p->info, p->sq, p->meta,
                    p->ncid, p->nvec,   p->nvec_tri, p->epp, p->eS, p->snorm, p->srow, p->scol,
                    p->geo, p->gip, p->fcol};
    for (void* q : ptrs)
        if (q) cudaFree(q);
    delete p;
}

int hxf_pairs_ties(const hxf_pairs* p, hxf_tie_record* out, int64_t capacity, int64_t* count) {
    HXF_TRY({
        if (!p) throw HxfError{HXF_EINVAL, "NULL pair tree"};
        if (count) *count = p->n_ovlp_ties;
        if (out)
            for (int64_t k = 0; k < capacity && k < (int64_t)p->ovlp_ties.size(); ++k) out[k] = p->ovlp_ties[k];
    })
}

int hxf_pairs_download(const hxf_pairs* p, int level, double* norm, double* rowsum, double* colsum,
                       uint8_t* pruned) {
    HXF_TRY({
        if (!p) throw HxfError{HXF_EINVAL, "NULL pairs"};
        const hxf_system* s = p->sys;
        if (level < 0 || level >= s->n_levels) throw HxfError{HXF_EINVAL, "level out of range"};
        set_device(s->device);
        const int64_t n = s->h_off[level + 1] - s->h_off[level];
        const int64_t o = s->node_off[level];
        std::vector<double> v(n * n);
        HXF_CUDA(cudaMemcpy(v.data(), p->norm + o, n * n * sizeof(double), cudaMemcpyDeviceToHost));
        for (int64_t k = 0; k < n * n; ++k) {
            if (pruned) pruned[k] = v[k] < 0.0;
            if (norm) norm[k] = v[k] < 0.0 ? 0.0 : v[k];
        }
        if (rowsum) HXF_CUDA(cudaMemcpy(rowsum, p->rowsum + o, n * n * sizeof(double), cudaMemcpyDeviceToHost));
        if (colsum) HXF_CUDA(cudaMemcpy(colsum, p->colsum + o, n * n * sizeof(double), cudaMemcpyDeviceToHost));
    })
}

int hxf_pairs_download_q(const hxf_pairs* p, double* q) {
    HXF_TRY({
        if (!p || !q) throw HxfError{HXF_EINVAL, "NULL argument"};
        const hxf_system* s = p->sys;
        set_device(s->device);
        const int ns = s->ns;
        std::vector<int> pi(p->n_pairs), pj(p->n_pairs);
        std::vector<double> qq(p->n_pairs);
        if (p->n_pairs) {
            HXF_CUDA(cudaMemcpy(pi.data(), p->pi, p->n_pairs * sizeof(int), cudaMemcpyDeviceToHost));
            HXF_CUDA(cudaMemcpy(pj.data(), p->pj, p->n_pairs * sizeof(int), cudaMemcpyDeviceToHost));
            HXF_CUDA(cudaMemcpy(qq.data(), p->q, p->n_pairs * sizeof(double), cudaMemcpyDeviceToHost));
        }
        for (int64_t k = 0; k < (int64_t)ns * ns; ++k) q[k] = -1.0;
        for (int64_t k = 0; k < p->n_pairs; ++k) q[(int64_t)pi[k] * ns + pj[k]] = qq[k];
    })
}

int hxf_pairs_overlap(const hxf_pairs* p, double* s_abs) {
    HXF_TRY({
        (void)p;
        (void)s_abs;
        throw HxfError{HXF_EINVAL, "hxf_pairs_overlap: not available in this build"};
    })
}

int hxf_density_build(hxf_system* s, const double* P, int P_on_device, double zero_drop, void* stream,
                      hxf_density** out) {
    HXF_TRY({
        if (!s || !P || !out) throw HxfError{HXF_EINVAL, "NULL argument"};
        set_device(s->device);
        hxf_density* d = new hxf_density();
        memset(d, 0, sizeof(*d));
        d->sys = s;
        d->device = s->device;
        d->zero_drop = zero_drop;
        try {
            trees_build_density(d, P, P_on_device, (cudaStream_t)stream);
        } catch (...) {
            hxf_density_destroy(d);
            throw;
        }
        *out = d;
    })
}

void hxf_density_destroy(hxf_density* d) {
    if (!d) return;
    cudaSetDevice(d->device);
    if (d->P) cudaFree(d->P);
    if (d->norm) cudaFree(d->norm);
    if (d->pmax) cudaFree(d->pmax);
    delete d;
}

int hxf_density_download(const hxf_density* d, int level, double* norm) {
    HXF_TRY({
        if (!d || !norm) throw HxfError{HXF_EINVAL, "NULL argument"};
        const hxf_system* s = d->sys;
        if (level < 0 || level >= s->n_levels) throw HxfError{HXF_EINVAL, "level out of range"};
        set_device(s->device);
        const int64_t n = s->h_off[level + 1] - s->h_off[level];
        HXF_CUDA(cudaMemcpy(norm, d->norm + s->node_off[level], n * n * sizeof(double), cudaMemcpyDeviceToHost));
    })
}

int hxf_density_download_pmax(const hxf_density* d, double* pmax) {
    HXF_TRY({
        if (!d || !pmax) throw HxfError{HXF_EINVAL, "NULL argument"};
        const hxf_system* s = d->sys;
        set_device(s->device);
        HXF_CUDA(cudaMemcpy(pmax, d->pmax, (size_t)s->ns * s->ns * sizeof(double), cudaMemcpyDeviceToHost));
    })
}

int hxf_exchange(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, const hxf_exchange_opts* opts,
                 double* K_out, hxf_counters* counters, void* stream) {
    HXF_TRY({
        if (!bra || !ket || !P || !opts || !counters) throw HxfError{HXF_EINVAL, "NULL argument"};
        set_device(bra->sys->device);
        memset(counters, 0, sizeof(*counters));
        exchange_run(bra, ket, P, opts, K_out, counters, (cudaStream_t)stream);
    })
}

int hxf_exchange_direct(hxf_pairs* pairs, hxf_density* P, const hxf_exchange_opts* opts, double* K_out,
                        hxf_counters* counters, void* stream) {
    HXF_TRY({
        if (!pairs || !P || !opts || !counters) throw HxfError{HXF_EINVAL, "NULL argument"};
        set_device(pairs->sys->device);
        memset(counters, 0, sizeof(*counters));
        direct_run(pairs, P, opts, K_out, counters, (cudaStream_t)stream);
    })
}

int hxf_frontier(hxf_pairs* bra, hxf_pairs* ket, hxf_density* P, double tau_2e, int mode, int symmetry,
                 int level, int64_t* n_tasks, double* cost, int64_t cost_capacity, void* stream) {
    HXF_TRY({
        if (!bra || !ket || !P || !n_tasks) throw HxfError{HXF_EINVAL, "NULL argument"};
        set_device(bra->sys->device);
        frontier_run(bra, ket, P, tau_2e, mode, symmetry == HXF_EIGHTFOLD ? 2 : (symmetry == HXF_FOURFOLD ? 1 : 0), level, n_tasks, cost,
                     cost_capacity, (cudaStream_t)stream);
    })
}

int hxf_last_timings(double* ms, int n) { return hxf_last_timings_impl(ms, n); }

int hxf_symmetrize(double* K_dev, int n, double tol, void* stream) {
    HXF_TRY({
        if (!K_dev || n < 0) throw HxfError{HXF_EINVAL, "bad arguments"};
        symmetrize_device(K_dev, n, tol, (cudaStream_t)stream);
    })
}

int hxf_fixed_to_double(const int64_t* Kfx, int64_t n2, int S, double* K, void* stream) {
    HXF_TRY({
        if ((!Kfx || !K) && n2 > 0) throw HxfError{HXF_EINVAL, "NULL argument"};
        if (n2 < 0) throw HxfError{HXF_EINVAL, "bad size"};
        fixed_to_double_impl(Kfx, n2, S, K, (cudaStream_t)stream);
    })
}

int hxf_fp64_peak(double* tflops, void* stream) {
    HXF_TRY({
        if (!tflops) throw HxfError{HXF_EINVAL, "NULL argument"};
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            throw HxfError{HXF_ECUDA, "no CUDA device available (libhxf has no CPU fallback)"};
        *tflops = fp64_peak((cudaStream_t)stream);
    })
}

int hxf_hilbert_order(const double* centers, int64_t n, int bits, int on_device, int64_t* perm,
                      uint64_t* keys, void* stream) {
    HXF_TRY({
        if (bits < 1 || bits > 20) throw HxfError{HXF_EINVAL, "bits_per_axis must be in [1, 20]"};
        if (n < 0 || n > INT32_MAX) throw HxfError{HXF_EINVAL, "bad shell count"};
        if (n > 0 && (!centers || !perm)) throw HxfError{HXF_EINVAL, "NULL argument"};
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw HxfError{HXF_ECUDA, "no CUDA device available (libhxf has no CPU fallback)"};
        cudaStream_t st = (cudaStream_t)stream;
        if (on_device) {
            hilbert_order_device(centers, n, bits, perm, keys, st);
        } else if (n > 0) {
            double* dc = (double*)hxf_cache_alloc(n * 3 * sizeof(double), st);
            int64_t* dp = (int64_t*)hxf_cache_alloc(n * sizeof(int64_t), st);
            uint64_t* dk = keys ? (uint64_t*)hxf_cache_alloc(n * sizeof(uint64_t), st) : nullptr;
            HXF_CUDA(cudaMemcpyAsync(dc, centers, n * 3 * sizeof(double), cudaMemcpyHostToDevice, st));
            hilbert_order_device(dc, n, bits, dp, dk, st);
            HXF_CUDA(cudaMemcpyAsync(perm, dp, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
            if (keys)
                HXF_CUDA(cudaMemcpyAsync(keys, dk, n * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
            HXF_CUDA(cudaStreamSynchronize(st));
            if (dk) hxf_cache_free(dk, st);
            hxf_cache_free(dp, st);
            hxf_cache_free(dc, st);
        }
    })
}

int hxf_partition_build(const int32_t* shell_nfunc, int64_t n_shells, int leaf_size,
                        int32_t* span_lo, int32_t* span_hi, int64_t span_capacity,
                        int64_t* level_off, int level_capacity, int64_t* n_spans, int* n_levels,
                        void* stream) {
    HXF_TRY({
        if (n_shells < 0 || n_shells >= INT32_MAX) throw HxfError{HXF_EINVAL, "bad shell count"};
        if ((n_shells > 0 && !shell_nfunc) || !span_lo || !span_hi || !level_off || !n_spans ||
            !n_levels)
            throw HxfError{HXF_EINVAL, "NULL argument"};
        int32_t big = 1;
        for (int64_t i = 0; i < n_shells; ++i) {
            if (shell_nfunc[i] < 1) throw HxfError{HXF_EINVAL, "shell with no functions"};
            big = std::max(big, shell_nfunc[i]);
        }
        if (leaf_size < big) throw HxfError{HXF_EINVAL, "leaf_size must be >= the largest shell"};
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
            throw HxfError{HXF_ECUDA, "no CUDA device available (libhxf has no CPU fallback)"};
        cudaStream_t st = (cudaStream_t)stream;
        std::vector<int64_t> off;
        std::vector<int32_t> lo, hi;
        if (n_shells == 0) {
            off = {0, 1};
            lo = {0};
            hi = {0};
        } else {
            int32_t* ds = (int32_t*)hxf_cache_alloc(n_shells * sizeof(int32_t), st);
            HXF_CUDA(cudaMemcpyAsync(ds, shell_nfunc, n_shells * sizeof(int32_t), cudaMemcpyHostToDevice, st));
            partition_build_device(ds, (int)n_shells, leaf_size, off, lo, hi, st);
            hxf_cache_free(ds, st);
        }
        *n_spans = (int64_t)lo.size();
        *n_levels = (int)off.size() - 1;
        if ((int64_t)lo.size() > span_capacity || (int64_t)off.size() > level_capacity)
            throw HxfError{HXF_EINVAL, "output capacity too small (sizes returned in n_spans, n_levels)"};
        memcpy(span_lo, lo.data(), lo.size() * sizeof(int32_t));
        memcpy(span_hi, hi.data(), hi.size() * sizeof(int32_t));
        memcpy(level_off, off.data(), off.size() * sizeof(int64_t));
    })
}

static void need_device() {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw HxfError{HXF_ECUDA, "no CUDA device available (libhxf has no CPU fallback)"};
}

int hxf_block_mask(const int64_t* K, int n, int bs, uint8_t* mask, void* stream) {
    HXF_TRY({
        if (n < 0 || bs < 1 || bs > 1024) throw HxfError{HXF_EINVAL, "bad size"};
        if (n > 0 && (!K || !mask)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        block_mask_device(K, n, bs, mask, (cudaStream_t)stream);
    })
}

int hxf_block_slots(const uint8_t* mask, int64_t n_tiles, int64_t* slot, int64_t* n_blocks, void* stream) {
    HXF_TRY({
        if (n_tiles < 0 || !n_blocks) throw HxfError{HXF_EINVAL, "bad arguments"};
        if (n_tiles > 0 && (!mask || !slot)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        *n_blocks = block_slots_device(mask, n_tiles, slot, (cudaStream_t)stream);
    })
}

int hxf_block_pack(const int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, int64_t* buf,
                   void* stream) {
    HXF_TRY({
        if (n < 0 || bs < 1 || bs > 1024) throw HxfError{HXF_EINVAL, "bad size"};
        if (n > 0 && (!K || !mask || !slot || !buf)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        block_move_device(const_cast<int64_t*>(K), n, bs, mask, slot, buf, true, (cudaStream_t)stream);
    })
}

int hxf_block_unpack(int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, const int64_t* buf,
                     void* stream) {
    HXF_TRY({
        if (n < 0 || bs < 1 || bs > 1024) throw HxfError{HXF_EINVAL, "bad size"};
        if (n > 0 && (!K || !mask || !slot || !buf)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        block_move_device(K, n, bs, mask, slot, const_cast<int64_t*>(buf), false, (cudaStream_t)stream);
    })
}

static void check_spans(int n, int nleaf, const void* flo, const void* fhi) {
    if (n < 0 || nleaf < 0 || nleaf > 32767) throw HxfError{HXF_EINVAL, "bad size"};
    if (nleaf > 0 && (!flo || !fhi)) throw HxfError{HXF_EINVAL, "NULL argument"};
}

int hxf_span_mask(const int64_t* K, int n, const int32_t* flo, const int32_t* fhi, int nleaf, uint8_t* mask,
                  void* stream) {
    HXF_TRY({
        check_spans(n, nleaf, flo, fhi);
        if (n > 0 && nleaf > 0 && (!K || !mask)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        span_mask_device(K, n, flo, fhi, nleaf, mask, (cudaStream_t)stream);
    })
}

int hxf_span_pack(const int64_t* K, int n, int row_base, const int32_t* flo, const int32_t* fhi, int nleaf,
                  int r0, int r1, const uint8_t* mask, const int64_t* off, int64_t off_base, int64_t* buf,
                  void* stream) {
    HXF_TRY({
        check_spans(n, nleaf, flo, fhi);
        if (r0 < 0 || r1 > nleaf || r0 > r1) throw HxfError{HXF_EINVAL, "bad row span range"};
        if (r1 > r0 && n > 0 && (!K || !mask || !off || !buf)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        span_move_device(const_cast<int64_t*>(K), n, row_base, flo, fhi, nleaf, r0, r1, mask, off, off_base, buf,
                         true, (cudaStream_t)stream);
    })
}

int hxf_span_unpack(int64_t* K, int n, int row_base, const int32_t* flo, const int32_t* fhi, int nleaf,
                    int r0, int r1, const uint8_t* mask, const int64_t* off, int64_t off_base, const int64_t* buf,
                    void* stream) {
    HXF_TRY({
        check_spans(n, nleaf, flo, fhi);
        if (r0 < 0 || r1 > nleaf || r0 > r1) throw HxfError{HXF_EINVAL, "bad row span range"};
        if (r1 > r0 && n > 0 && (!K || !mask || !off || !buf)) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        span_move_device(K, n, row_base, flo, fhi, nleaf, r0, r1, mask, off, off_base, const_cast<int64_t*>(buf),
                         false, (cudaStream_t)stream);
    })
}

int hxf_fixed_fold(int64_t* K, int n, void* stream) {
    HXF_TRY({
        if (n < 0) throw HxfError{HXF_EINVAL, "bad size"};
        if (n > 0 && !K) throw HxfError{HXF_EINVAL, "NULL argument"};
        need_device();
        fold_fixed_device(K, n, (cudaStream_t)stream);
    })
}

int hxf_scratch_release(int64_t* bytes) {
    HXF_TRY({
        int dev = 0;
        cudaGetDevice(&dev);
        HXF_CUDA(cudaDeviceSynchronize());
        ScratchCache& c = scratch_cache();
        int64_t total = 0;
        {
            std::lock_guard<std::mutex> g(c.mu);
            for (auto& kv : c.free_lists) {
                if (std::get<0>(kv.first) != dev) continue;
                for (void* q : kv.second) {
                    cudaFree(q);
                    c.dev_of.erase(q);
                    total += (int64_t)std::get<2>(kv.first);
                }
                kv.second.clear();
            }
        }
        if (bytes) *bytes = total;
    })
}

int hxf_launch_count(int64_t* n) {
    HXF_TRY({
        if (!n) throw HxfError{HXF_EINVAL, "NULL argument"};
        *n = g_launches.load();
    })
}

}  // extern "C"
