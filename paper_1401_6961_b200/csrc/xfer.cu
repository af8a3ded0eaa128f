// Host <-> device transfers of the drop-in boundary's big arrays (the density P in,
// K out: n^2 doubles, 6.6 GB each at BASELINE config 5) when the caller's buffers are
// ordinary pageable memory, as a reference caller's numpy arrays are
// (build_matrix_tree(P), quadtree.py:198; K returned by build_exchange_*,
// exchange_naive.py:200-240).  A plain cudaMemcpy from pageable memory stages through
// one driver thread (~5 GB/s measured: 2.6 s of a 9.8 s end-to-end c5 build).  Here a
// few worker threads each move their share of the array in 16 MB pieces through their
// own pair of pinned buffers on their own stream: the host memcpy of one piece overlaps
// the DMA of the previous one, and the workers' memcpys (and the page faults of a fresh
// destination) run in parallel.  Pinned buffers and streams are created once per device.
#include <algorithm>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "hxf_internal.cuh"

namespace {

constexpr size_t PIECE = 16u << 20;          // bytes per pinned buffer
constexpr size_t STAGED_MIN = 64u << 20;     // below this a plain copy is used
constexpr int MAX_WORKERS = 16;

struct Worker {
    cudaStream_t stream = nullptr;
    char* pin[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
};

struct Pool {
    int device = -1;
    std::vector<Worker> w;
};

std::mutex g_mu;
std::vector<Pool> g_pools;

int worker_count() {
    static const int n = [] {
        if (const char* e = getenv("HXF_XFER_THREADS")) return std::max(1, std::min(MAX_WORKERS, atoi(e)));
        const unsigned hc = std::thread::hardware_concurrency();
        return (int)std::max(1u, std::min<unsigned>(MAX_WORKERS, hc ? hc / 2 : 4));
    }();
    return n;
}

// the calling thread holds g_mu for the whole transfer (one staged transfer at a time per process)
Pool& pool_for(int device) {
    for (Pool& p : g_pools)
        if (p.device == device) return p;
    g_pools.emplace_back();
    Pool& p = g_pools.back();
    p.device = device;
    p.w.resize(worker_count());
    for (Worker& w : p.w) {
        HXF_CUDA(cudaStreamCreateWithFlags(&w.stream, cudaStreamNonBlocking));
        for (int b = 0; b < 2; ++b) {
            HXF_CUDA(cudaHostAlloc((void**)&w.pin[b], PIECE, cudaHostAllocDefault));
            HXF_CUDA(cudaEventCreateWithFlags(&w.ev[b], cudaEventDisableTiming));
        }
    }
    return p;
}

// worker k moves the pieces k, k + W, k + 2W, ... of [0, bytes)
void run_worker(int device, Worker* w, int k, int W, char* dev, char* host, size_t bytes, bool to_device,
                cudaError_t* err) {
    cudaError_t e = cudaSetDevice(device);
    const size_t npiece = (bytes + PIECE - 1) / PIECE;
    size_t pending_off[2] = {0, 0}, pending_len[2] = {0, 0};
    int it = 0;
    for (size_t p = k; p < npiece && e == cudaSuccess; p += W, ++it) {
        const int b = it & 1;
        const size_t off = p * PIECE, len = std::min(PIECE, bytes - off);
        if (to_device) {
            if (it >= 2) e = cudaEventSynchronize(w->ev[b]);      // the buffer's previous DMA is done
            if (e != cudaSuccess) break;
            memcpy(w->pin[b], host + off, len);
            e = cudaMemcpyAsync(dev + off, w->pin[b], len, cudaMemcpyHostToDevice, w->stream);
            if (e == cudaSuccess) e = cudaEventRecord(w->ev[b], w->stream);
        } else {
            // drain the buffer's previous piece to the host array, then refill it
            if (it >= 2) {
                e = cudaEventSynchronize(w->ev[b]);
                if (e != cudaSuccess) break;
                memcpy(host + pending_off[b], w->pin[b], pending_len[b]);
            }
            e = cudaMemcpyAsync(w->pin[b], dev + off, len, cudaMemcpyDeviceToHost, w->stream);
            if (e == cudaSuccess) e = cudaEventRecord(w->ev[b], w->stream);
            pending_off[b] = off;
            pending_len[b] = len;
        }
    }
    if (!to_device && e == cudaSuccess) {
        for (int j = 0; j < 2 && j < it; ++j) {   // oldest first
            const int b = (it - std::min(it, 2) + j) & 1;
            e = cudaEventSynchronize(w->ev[b]);
            if (e != cudaSuccess) break;
            memcpy(host + pending_off[b], w->pin[b], pending_len[b]);
        }
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(w->stream);
    *err = e;
}

void staged(void* dev, void* host, size_t bytes, bool to_device, cudaStream_t st) {
    int device = 0;
    HXF_CUDA(cudaGetDevice(&device));
    std::lock_guard<std::mutex> lock(g_mu);
    Pool& pool = pool_for(device);
    const int W = (int)pool.w.size();
    // order against the caller's stream: the workers start after everything queued on st
    cudaEvent_t ready;
    HXF_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    HXF_CUDA(cudaEventRecord(ready, st));
    for (Worker& w : pool.w) HXF_CUDA(cudaStreamWaitEvent(w.stream, ready, 0));
    std::vector<std::thread> th;
    std::vector<cudaError_t> errs(W, cudaSuccess);
    for (int k = 0; k < W; ++k)
        th.emplace_back(run_worker, device, &pool.w[k], k, W, (char*)dev, (char*)host, bytes, to_device, &errs[k]);
    for (std::thread& t : th) t.join();
    cudaEventDestroy(ready);
    for (cudaError_t e : errs) HXF_CUDA(e);
    // every worker synchronised its stream: the data is in place; later work on st is ordered after this call
}

}  // namespace

// P (or any large host array) to the device, ordered after the work queued on st; returns when done
void xfer_to_device(void* dst_dev, const void* src_host, size_t bytes, cudaStream_t st) {
    static const bool off = getenv("HXF_XFER_PLAIN") != nullptr;   // A/B: the plain pageable copy
    if (bytes < STAGED_MIN || off) {
        HXF_CUDA(cudaMemcpyAsync(dst_dev, src_host, bytes, cudaMemcpyHostToDevice, st));
        return;
    }
    NvtxRange r("hxf: staged H2D");
    staged(dst_dev, const_cast<void*>(src_host), bytes, true, st);
}

// K (or any large device array) to a host array, ordered after the work queued on st; returns when done
void xfer_to_host(void* dst_host, const void* src_dev, size_t bytes, cudaStream_t st) {
    static const bool off = getenv("HXF_XFER_PLAIN") != nullptr;
    if (bytes < STAGED_MIN || off) {
        HXF_CUDA(cudaMemcpyAsync(dst_host, src_dev, bytes, cudaMemcpyDeviceToHost, st));
        return;
    }
    NvtxRange r("hxf: staged D2H");
    staged(const_cast<void*>(src_dev), dst_host, bytes, false, st);
}
