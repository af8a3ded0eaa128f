// Block-sparse K for the multi-GPU reduction (first part).
//
// A shard's K is its n x n int64 fixed-point accumulator (hxf_exchange_opts.K_fixed).
// Exchange K is block sparse at c5 scale (|K_ij| decays with the distance of i and j),
// so instead of all-reducing n^2 int64 the ranks
//   1. flag the bs x bs tiles holding any nonzero (hxf_block_mask),
//   2. OR the flags over the job (a small uint8 all-reduce, max),
//   3. number the flagged tiles (hxf_block_slots: exclusive scan, count to host),
//   4. pack those tiles into a dense buffer (hxf_block_pack), all-reduce it (int64
//      sum: exact), and unpack (hxf_block_unpack).
// A tile flagged by no rank is zero on every rank, so it needs no traffic and the
// unpacked K is bitwise the dense all-reduce.  Tiles are row-major, edge tiles
// zero-padded.  Mask / pack / unpack are HBM-bound streaming passes: one CTA per
// tile, 64-bit loads coalesced along K rows; the mask pass stops reading a tile
// at its first nonzero chunk.

#include <cub/cub.cuh>

#include "hxf_internal.cuh"

namespace {

// one block per tile: any nonzero in rows [ti*bs, ..) x cols [tj*bs, ..)
__global__ void k_block_mask(const int64_t* __restrict__ K, int n, int bs, int nb, bool v16,
                             uint8_t* __restrict__ mask) {
    const int64_t t = blockIdx.x;
    const int ti = (int)(t / nb), tj = (int)(t % nb);
    const int r0 = ti * bs, c0 = tj * bs;
    const int rn = min(bs, n - r0), cn = min(bs, n - c0);
    // chunks of 4 loads per thread, the block leaves at the first chunk holding a
    // nonzero: a nonzero tile (55 % at c5) is usually decided by its first chunk,
    // so only the zero tiles are read in full
    const int total = rn * cn;
    int any = 0;
    if (v16) {  // even n and bs, 16-byte aligned K: 16-byte pairs, 8 KB chunks as below
        const int half = total / 2, cp = cn / 2;
        for (int base = 0; base < half; base += 2 * blockDim.x) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
                const int e = base + u * blockDim.x + threadIdx.x;
                if (e < half) {
                    const int r = e / cp, c = 2 * (e - r * cp);
                    const longlong2 v = __ldcs(reinterpret_cast<const longlong2*>(
                        K + (int64_t)(r0 + r) * n + c0 + c));
                    any |= (v.x | v.y) != 0;
                }
            }
            if (__syncthreads_or(any)) {
                any = 1;
                break;
            }
        }
        if (threadIdx.x == 0) mask[t] = (uint8_t)any;
        return;
    }
    for (int base = 0; base < total; base += 4 * blockDim.x) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = base + u * blockDim.x + threadIdx.x;
            if (e < total) {
                const int r = e / cn, c = e - r * cn;
                any |= __ldcs(K + (int64_t)(r0 + r) * n + c0 + c) != 0;
            }
        }
        if (__syncthreads_or(any)) {
            any = 1;
            break;
        }
    }
    if (threadIdx.x == 0) mask[t] = (uint8_t)any;
}

__global__ void k_mask_to_int(const uint8_t* __restrict__ m, int64_t nt, int64_t* __restrict__ v) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nt; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = m[i] ? 1 : 0;
}

template <bool PACK>
__global__ void k_block_move(int64_t* __restrict__ K, int n, int bs, int nb, bool v16,
                             const uint8_t* __restrict__ mask, const int64_t* __restrict__ slot,
                             int64_t* __restrict__ buf) {
    const int64_t t = blockIdx.x;
    if (!mask[t]) return;
    const int ti = (int)(t / nb), tj = (int)(t % nb);
    const int r0 = ti * bs, c0 = tj * bs;
    int64_t* b = buf + slot[t] * (int64_t)bs * bs;
    if (v16) {  // even n and bs, 16-byte aligned K and buf: aligned pairs along a row
        longlong2* b2 = reinterpret_cast<longlong2*>(b);
        for (int e = threadIdx.x; e < bs * bs / 2; e += blockDim.x) {
            const int r = (2 * e) / bs, c = 2 * e - r * bs;
            const bool in = r0 + r < n && c0 + c < n;  // c even, n even: c + 1 < n too
            longlong2* k2 = reinterpret_cast<longlong2*>(K + (int64_t)(r0 + r) * n + c0 + c);
            if (PACK) {
                b2[e] = in ? __ldcs(k2) : make_longlong2(0, 0);
            } else if (in) {
                __stcs(k2, b2[e]);
            }
        }
        return;
    }
    for (int e = threadIdx.x; e < bs * bs; e += blockDim.x) {
        const int r = e / bs, c = e % bs;
        const bool in = r0 + r < n && c0 + c < n;
        if (PACK) {
            b[e] = in ? K[(int64_t)(r0 + r) * n + c0 + c] : 0;
        } else if (in) {
            K[(int64_t)(r0 + r) * n + c0 + c] = b[e];
        }
    }
}

// 16-byte accesses need even n and bs (pairs never straddle a row or tile edge)
// and 16-byte aligned base pointers
bool use_v16(int n, int bs, const void* a, const void* b) {
    return ((n | bs) & 1) == 0 && ((((uintptr_t)a) | ((uintptr_t)b)) & 15) == 0;
}

// one CTA per tile: the grid must fit the launch limit
void check_tiles(int64_t nt) {
    if (nt > 0x7fffffffll)
        throw HxfError{HXF_EINVAL, "block size too small for n: more than 2^31-1 tiles"};
}

}  // namespace

void block_mask_device(const int64_t* K, int n, int bs, uint8_t* mask, cudaStream_t st) {
    const int nb = (n + bs - 1) / bs;
    const int64_t nt = (int64_t)nb * nb;
    if (nt == 0) return;
    check_tiles(nt);
    { k_block_mask<<<(unsigned)nt, 256, 0, st>>>(K, n, bs, nb, use_v16(n, bs, K, K), mask); note_launch(); }
    HXF_CUDA(cudaGetLastError());
}

int64_t block_slots_device(const uint8_t* mask, int64_t nt, int64_t* slot, cudaStream_t st) {
    if (nt == 0) return 0;
    int64_t* v = (int64_t*)hxf_cache_alloc((nt + 1) * sizeof(int64_t), st);
    HXF_CUDA(cudaMemsetAsync(v + nt, 0, sizeof(int64_t), st));
    { k_mask_to_int<<<(unsigned)std::min<int64_t>((nt + 255) / 256, 148 * 8), 256, 0, st>>>(mask, nt, v); note_launch(); }
    size_t tb = 0;
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, v, slot, nt + 1, st));
    void* tmp = hxf_cache_alloc(tb ? tb : 1, st);
    HXF_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, v, slot, nt + 1, st));  // slot[nt] = count
    note_launch();
    int64_t count = 0;
    HXF_CUDA(cudaMemcpyAsync(&count, slot + nt, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    HXF_CUDA(cudaStreamSynchronize(st));
    hxf_cache_free(tmp, st);
    hxf_cache_free(v, st);
    return count;
}

void block_move_device(int64_t* K, int n, int bs, const uint8_t* mask, const int64_t* slot, int64_t* buf,
                       bool pack, cudaStream_t st) {
    const int nb = (n + bs - 1) / bs;
    const int64_t nt = (int64_t)nb * nb;
    if (nt == 0) return;
    check_tiles(nt);
    const bool v16 = use_v16(n, bs, K, buf);
    if (pack) {
        k_block_move<true><<<(unsigned)nt, 256, 0, st>>>(K, n, bs, nb, v16, mask, slot, buf);
    } else {
        k_block_move<false><<<(unsigned)nt, 256, 0, st>>>(K, n, bs, nb, v16, mask, slot, buf);
    }
    note_launch();
    HXF_CUDA(cudaGetLastError());
}

// ---------------------------------------------------------------------------
// K quadtree leaves (second part; PAPER.md:174-198 treats K as a
// quadtree over the same index bisection as P).  A leaf tile (r, c) is the block
// rows [flo[r], fhi[r]) x cols [flo[c], fhi[c]) of the partition's leaf spans r, c
// (ragged: spans hold different function counts).  Occupancy of the leaf tiles is
// the quadtree's bottom level; the host ORs it up the span tree.  Pack / unpack move
// the flagged tiles between K (or a row block of K) and one dense buffer in tile
// row-major order, each tile row-major inside, at the element offsets the caller
// scanned from the occupancy: a rank's rows are one contiguous slice of the buffer,
// which is what the reduce-scatter of distributed.reduce_scatter_quadtree sends.
// One CTA per leaf row span: whole K rows are read / written coalesced.

namespace {

__global__ void k_span_index(const int* __restrict__ flo, const int* __restrict__ fhi, int nleaf,
                             int* __restrict__ leaf_of_fn) {
    const int r = blockIdx.x;
    if (r >= nleaf) return;
    for (int f = flo[r] + threadIdx.x; f < fhi[r]; f += blockDim.x) leaf_of_fn[f] = r;
}

__global__ void __launch_bounds__(256) k_span_mask(const int64_t* __restrict__ K, int n, const int* __restrict__ flo,
                                                   const int* __restrict__ fhi, int nleaf,
                                                   const int* __restrict__ leaf_of_fn, uint8_t* __restrict__ mask) {
    extern __shared__ unsigned s_flag[];   // one bit per column span
    const int r = blockIdx.x, words = (nleaf + 31) / 32;
    for (int i = threadIdx.x; i < words; i += blockDim.x) s_flag[i] = 0u;
    __syncthreads();
    for (int row = flo[r]; row < fhi[r]; ++row) {
        const int64_t* kr = K + (int64_t)row * n;
        for (int c = threadIdx.x; c < n; c += blockDim.x)
            if (__ldcs(kr + c) != 0) {
                const int lc = leaf_of_fn[c];
                atomicOr(&s_flag[lc >> 5], 1u << (lc & 31));
            }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < nleaf; c += blockDim.x)
        mask[(int64_t)r * nleaf + c] = (uint8_t)((s_flag[c >> 5] >> (c & 31)) & 1u);
}

// K addresses rows relative to row_base (K may be a row block of the matrix)
template <bool PACK>
__global__ void __launch_bounds__(256) k_span_move(int64_t* __restrict__ K, int n, int row_base,
                                                   const int* __restrict__ flo, const int* __restrict__ fhi, int nleaf,
                                                   int r0, const int* __restrict__ leaf_of_fn,
                                                   const uint8_t* __restrict__ mask, const int64_t* __restrict__ off,
                                                   int64_t off_base, int64_t* __restrict__ buf) {
    const int r = r0 + blockIdx.x;
    const uint8_t* mr = mask + (int64_t)r * nleaf;
    const int64_t* orow = off + (int64_t)r * nleaf;
    for (int row = flo[r]; row < fhi[r]; ++row) {
        int64_t* kr = K + (int64_t)(row - row_base) * n;
        const int dr = row - flo[r];
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            const int lc = leaf_of_fn[c];
            if (!mr[lc]) continue;
            const int w = fhi[lc] - flo[lc];
            int64_t* b = buf + (orow[lc] - off_base) + (int64_t)dr * w + (c - flo[lc]);
            if (PACK) *b = kr[c];
            else kr[c] = *b;
        }
    }
}

}  // namespace

void span_index_device(const int* flo, const int* fhi, int nleaf, int* leaf_of_fn, cudaStream_t st) {
    if (nleaf <= 0) return;
    { k_span_index<<<nleaf, 32, 0, st>>>(flo, fhi, nleaf, leaf_of_fn); note_launch(); }
    HXF_CUDA(cudaGetLastError());
}

void span_mask_device(const int64_t* K, int n, const int* flo, const int* fhi, int nleaf, uint8_t* mask,
                      cudaStream_t st) {
    if (nleaf <= 0 || n <= 0) return;
    int* lof = (int*)hxf_cache_alloc((size_t)n * sizeof(int), st);
    span_index_device(flo, fhi, nleaf, lof, st);
    const size_t smem = (size_t)((nleaf + 31) / 32) * sizeof(unsigned);
    { k_span_mask<<<nleaf, 256, smem, st>>>(K, n, flo, fhi, nleaf, lof, mask); note_launch(); }
    HXF_CUDA(cudaGetLastError());
    hxf_cache_free(lof, st);
}

void span_move_device(int64_t* K, int n, int row_base, const int* flo, const int* fhi, int nleaf, int r0, int r1,
                      const uint8_t* mask, const int64_t* off, int64_t off_base, int64_t* buf, bool pack,
                      cudaStream_t st) {
    if (r1 <= r0 || n <= 0) return;
    int* lof = (int*)hxf_cache_alloc((size_t)n * sizeof(int), st);
    span_index_device(flo, fhi, nleaf, lof, st);
    if (pack) k_span_move<true><<<r1 - r0, 256, 0, st>>>(K, n, row_base, flo, fhi, nleaf, r0, lof, mask, off, off_base, buf);
    else k_span_move<false><<<r1 - r0, 256, 0, st>>>(K, n, row_base, flo, fhi, nleaf, r0, lof, mask, off, off_base, buf);
    note_launch();
    HXF_CUDA(cudaGetLastError());
    hxf_cache_free(lof, st);
}
