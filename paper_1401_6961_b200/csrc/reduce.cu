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
