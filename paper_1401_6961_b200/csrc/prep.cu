// Device input preparation (first part): the 3-D Hilbert
// reordering of shells.  Restates basis.py:275-331 of the reference:
//   - lattice point per shell: rint((c - lo) / extent * side) per axis, side =
//     2^bits - 1, axis left at 0 when its extent is 0 (basis.py:309-325);
//   - Skilling's transposed-bits Hilbert index (basis.py:275-306);
//   - stable argsort of the keys (basis.py:326-327).
// Every float64 step is one correctly rounded IEEE operation, as numpy does it
// (no FMA contraction), and np.rint is round-half-even like rint(), so the
// lattice and the keys are bitwise the host's; cub's LSD radix sort is stable,
// so the permutation is numpy's kind="stable" argsort.
//
// Layout: centers are n x 3 float64 row-major in HBM (24 B per shell read twice:
// once by the extent reduction, once by the key kernel); keys are uint64
// (3 * bits <= 60 significant bits), the permutation int64.  A setup pass of a
// few hundred kB at c5: launch-latency bound, grid sized in multiples of the SMs.

#include <cub/cub.cuh>

#include "hxf_internal.cuh"

namespace {

// per-axis min and max (exact: no rounding in a min/max); one block per axis
// keeps the result independent of the grid (deterministic, no atomics).
__global__ void k_extent(const double* __restrict__ c, int64_t n, double* __restrict__ lo_ext) {
    const int ax = blockIdx.x;
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
        double v = c[3 * i + ax];
        lo = fmin(lo, v);
        hi = fmax(hi, v);
    }
    typedef cub::BlockReduce<double, 1024> R;
    __shared__ typename R::TempStorage ts;
    double blo = R(ts).Reduce(lo, [](double a, double b) { return fmin(a, b); });
    __syncthreads();
    double bhi = R(ts).Reduce(hi, [](double a, double b) { return fmax(a, b); });
    if (threadIdx.x == 0) {
        lo_ext[ax] = blo;
        lo_ext[3 + ax] = __dsub_rn(bhi, blo);  // extent = max - lo (basis.py:318)
    }
}

// Skilling transposed-bits Hilbert index of one lattice point (basis.py:275-306)
__device__ __forceinline__ uint64_t hilbert_key(uint32_t x0, uint32_t x1, uint32_t x2, int bits) {
    uint32_t x[3] = {x0, x1, x2};
    const uint32_t m = 1u << (bits - 1);
    for (uint32_t q = m; q > 1; q >>= 1) {
        const uint32_t p = q - 1;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            if (x[i] & q) {
                x[0] ^= p;
            } else {
                uint32_t t = (x[0] ^ x[i]) & p;
                x[0] ^= t;
                x[i] ^= t;
            }
        }
    }
    x[1] ^= x[0];
    x[2] ^= x[1];
    uint32_t t = 0;
    for (uint32_t q = m; q > 1; q >>= 1)
        if (x[2] & q) t ^= q - 1;
    x[0] ^= t;
    x[1] ^= t;
    x[2] ^= t;
    uint64_t h = 0;
    for (int b = bits - 1; b >= 0; --b) {
#pragma unroll
        for (int i = 0; i < 3; ++i) h = (h << 1) | ((x[i] >> b) & 1u);
    }
    return h;
}

__global__ void k_hilbert_keys(const double* __restrict__ c, int64_t n, int bits,
                               const double* __restrict__ lo_ext, uint64_t* __restrict__ keys,
                               int64_t* __restrict__ idx) {
    const double side = (double)((1u << bits) - 1u);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t l[3];
#pragma unroll
        for (int ax = 0; ax < 3; ++ax) {
            const double ext = lo_ext[3 + ax];
            l[ax] = 0;
            if (ext > 0.0)  // basis.py:323-324
                l[ax] = (uint32_t)rint(__dmul_rn(__ddiv_rn(__dsub_rn(c[3 * i + ax], lo_ext[ax]), ext), side));
        }
        keys[i] = hilbert_key(l[0], l[1], l[2], bits);
        idx[i] = i;
    }
}

}  // namespace

void hilbert_order_device(const double* centers, int64_t n, int bits, int64_t* perm,
                          uint64_t* keys_out, cudaStream_t st) {
    if (n == 0) return;
    int dev = 0, sms = 0;
    HXF_CUDA(cudaGetDevice(&dev));
    HXF_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    double* lo_ext = (double*)hxf_cache_alloc(6 * sizeof(double), st);
    uint64_t* k0 = (uint64_t*)hxf_cache_alloc(n * sizeof(uint64_t), st);
    uint64_t* k1 = keys_out ? keys_out : (uint64_t*)hxf_cache_alloc(n * sizeof(uint64_t), st);
    int64_t* i0 = (int64_t*)hxf_cache_alloc(n * sizeof(int64_t), st);
    { k_extent<<<3, 1024, 0, st>>>(centers, n, lo_ext); note_launch(); }
    const int64_t want = (n + 255) / 256;
    const int grid = (int)std::min<int64_t>(want, (int64_t)sms * 8);
    { k_hilbert_keys<<<grid, 256, 0, st>>>(centers, n, bits, lo_ext, k0, i0); note_launch(); }
    size_t tb = 0;
    HXF_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0, k1, i0, perm, (int)n, 0, 3 * bits, st));
    void* tmp = hxf_cache_alloc(tb ? tb : 1, st);
    HXF_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, k0, k1, i0, perm, (int)n, 0, 3 * bits, st));
    note_launch();
    HXF_CUDA(cudaGetLastError());
    hxf_cache_free(tmp, st);
    hxf_cache_free(i0, st);
    if (!keys_out) hxf_cache_free(k1, st);
    hxf_cache_free(k0, st);
    hxf_cache_free(lo_ext, st);
}

// ------------------------------------------------------------------ partition
// Level-synchronous device restatement of build_partition (quadtree.py:90-113):
// a span with more than leaf_size functions splits at the shell boundary b in
// (lo, hi) minimising |cum[b] - mid|, mid = (fn_lo + fn_hi) / 2, ties to the
// smaller b (np.argmin takes the first); a leaf repeats at the next level
// (Partition.levels).  cum is strictly increasing, so |cum[b] - mid| is unimodal
// in b and one binary search per span replaces the reference's scan over all
// candidates.  Every value is an integer below 2^53: the double compares are exact.

namespace {

__global__ void k_split(const int64_t* __restrict__ cum, const int32_t* __restrict__ lo,
                        const int32_t* __restrict__ hi, int m, int leaf,
                        int32_t* __restrict__ nchild, int32_t* __restrict__ bsplit) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int a = lo[s], z = hi[s];
    const int64_t fl = cum[a], fh = cum[z];
    if (fh - fl <= leaf) {
        nchild[s] = 1;
        bsplit[s] = -1;
        return;
    }
    const double mid = (double)(fl + fh) / 2.0;
    int l = a + 1, r = z - 1;  // first b in [a+1, z-1] with cum[b] >= mid, else z-1
    while (l < r) {
        const int c = (l + r) >> 1;
        if ((double)cum[c] >= mid) r = c; else l = c + 1;
    }
    int b = l;
    if (b - 1 >= a + 1 && fabs((double)cum[b - 1] - mid) <= fabs((double)cum[b] - mid)) b = b - 1;
    nchild[s] = 2;
    bsplit[s] = b;
}

__global__ void k_emit(const int32_t* __restrict__ lo, const int32_t* __restrict__ hi, int m,
                       const int32_t* __restrict__ off, const int32_t* __restrict__ bsplit,
                       int32_t* __restrict__ nlo, int32_t* __restrict__ nhi) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= m) return;
    const int o = off[s], b = bsplit[s];
    if (b < 0) {
        nlo[o] = lo[s];
        nhi[o] = hi[s];
    } else {
        nlo[o] = lo[s];
        nhi[o] = b;
        nlo[o + 1] = b;
        nhi[o + 1] = hi[s];
    }
}

}  // namespace

// sizes: device int32 function counts per shell.  Returns the level tables on
// the host: level k's spans are [level_off[k], level_off[k+1]) of span_lo/hi.
void partition_build_device(const int32_t* sizes, int n, int leaf, std::vector<int64_t>& level_off,
                            std::vector<int32_t>& span_lo, std::vector<int32_t>& span_hi,
                            cudaStream_t st) {
    int64_t* cum = (int64_t*)hxf_cache_alloc((n + 1) * sizeof(int64_t), st);
    HXF_CUDA(cudaMemsetAsync(cum, 0, sizeof(int64_t), st));
    size_t tb = 0;
    HXF_CUDA(cub::DeviceScan::InclusiveSum(nullptr, tb, sizes, cum + 1, n, st));
    // a level holds at most n spans (spans partition the shells), so one scratch
    // size serves every level's scan
    size_t tb2 = 0;
    int32_t* dummy = nullptr;
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb2, dummy, dummy, n + 1, st));
    tb = std::max(tb, tb2);
    void* tmp = hxf_cache_alloc(tb ? tb : 1, st);
    HXF_CUDA(cub::DeviceScan::InclusiveSum(tmp, tb, sizes, cum + 1, n, st));
    note_launch();
    int32_t* lo = (int32_t*)hxf_cache_alloc((n + 1) * sizeof(int32_t), st);
    int32_t* hi = (int32_t*)hxf_cache_alloc((n + 1) * sizeof(int32_t), st);
    int32_t* nlo = (int32_t*)hxf_cache_alloc((n + 1) * sizeof(int32_t), st);
    int32_t* nhi = (int32_t*)hxf_cache_alloc((n + 1) * sizeof(int32_t), st);
    int32_t* nch = (int32_t*)hxf_cache_alloc((n + 2) * sizeof(int32_t), st);
    int32_t* off = (int32_t*)hxf_cache_alloc((n + 2) * sizeof(int32_t), st);
    int32_t* bs = (int32_t*)hxf_cache_alloc((n + 1) * sizeof(int32_t), st);
    const int32_t root[2] = {0, n};
    HXF_CUDA(cudaMemcpyAsync(lo, &root[0], sizeof(int32_t), cudaMemcpyHostToDevice, st));
    HXF_CUDA(cudaMemcpyAsync(hi, &root[1], sizeof(int32_t), cudaMemcpyHostToDevice, st));
    level_off.assign(1, 0);
    span_lo.clear();
    span_hi.clear();
    int m = 1;
    for (;;) {
        const size_t base = span_lo.size();
        span_lo.resize(base + m);
        span_hi.resize(base + m);
        HXF_CUDA(cudaMemcpyAsync(span_lo.data() + base, lo, m * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaMemcpyAsync(span_hi.data() + base, hi, m * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        level_off.push_back((int64_t)base + m);
        const int g = (m + 255) / 256;
        { k_split<<<g, 256, 0, st>>>(cum, lo, hi, m, leaf, nch, bs); note_launch(); }
        HXF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, nch, off, m + 1, st));  // off[m] = total
        note_launch();
        int32_t total = 0;
        HXF_CUDA(cudaMemcpyAsync(&total, off + m, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
        HXF_CUDA(cudaStreamSynchronize(st));
        if (total == m) break;  // every span a leaf: this level is the last
        { k_emit<<<g, 256, 0, st>>>(lo, hi, m, off, bs, nlo, nhi); note_launch(); }
        std::swap(lo, nlo);
        std::swap(hi, nhi);
        m = total;
    }
    HXF_CUDA(cudaGetLastError());
    for (void* p : {(void*)cum, tmp, (void*)lo, (void*)hi, (void*)nlo, (void*)nhi, (void*)nch,
                    (void*)off, (void*)bs})
        hxf_cache_free(p, st);
}
