// host_pipeline.h -- the end-to-end (host buffer) side of the library: the
// chunked H2D -> scan -> D2H pipeline behind ps_scan_host / ps_scan_batched_host.
//
// The reference's users hand `sequential_inclusive_scan` a plain numpy array
// (core.py:118-126) and get it back scanned in place.  On the GPU that is a
// PCIe round trip, so the pipeline overlaps, chunk by chunk, the host->device
// copy of chunk k+1, the scan of chunk k and the device->host copy of chunk
// k-1 (three streams, NSLOT device slots).  Page-locked host memory is DMA'd
// directly.  Pageable memory cannot be (the driver would stage it through its
// own small pinned buffer and serialise), so it goes through a ring of pinned
// bounce buffers: a pool of host copy threads fills the bounce slot of chunk
// k+1 and drains the one of chunk k-2 while the DMA engines move chunk k.
//
// Host-only C++ (no device code); included by prefixscan_b200.cu.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <immintrin.h>
#include <cstdint>
#include <cstring>
#include <deque>
#include <mutex>
#include <thread>
#include <vector>

namespace ps {
namespace host {

constexpr int NSLOT = 3;                 // device (and bounce) slots in flight
constexpr size_t COPY_PIECE = 1u << 20;  // host memcpy granularity across the pool

// Host copy with streaming (non-temporal) stores: the destination -- a bounce
// slot the DMA engine reads next, or the caller's output array -- is not read
// back by this thread, so writing around the caches saves the read-for-
// ownership of every destination line (a third of the host memory traffic of
// a plain memcpy).  The staging path is bound by host memory bandwidth
// (profiles/r02_e2e.md), so this is its main lever.
__attribute__((target("avx2"))) inline void stream_copy_avx2(char *dst, const char *src, size_t n) {
    const size_t head = (32 - ((uintptr_t)dst & 31)) & 31;
    if (n < head + 256) {
        std::memcpy(dst, src, n);
        return;
    }
    std::memcpy(dst, src, head);
    dst += head, src += head, n -= head;
    size_t i = 0;
    for (; i + 128 <= n; i += 128) {
        __m256i a = _mm256_loadu_si256((const __m256i *)(src + i));
        __m256i b = _mm256_loadu_si256((const __m256i *)(src + i + 32));
        __m256i c = _mm256_loadu_si256((const __m256i *)(src + i + 64));
        __m256i d = _mm256_loadu_si256((const __m256i *)(src + i + 96));
        _mm256_stream_si256((__m256i *)(dst + i), a);
        _mm256_stream_si256((__m256i *)(dst + i + 32), b);
        _mm256_stream_si256((__m256i *)(dst + i + 64), c);
        _mm256_stream_si256((__m256i *)(dst + i + 96), d);
    }
    _mm_sfence();
    std::memcpy(dst + i, src + i, n - i);
}

inline void host_copy(char *dst, const char *src, size_t n) {
    static const bool avx2 = __builtin_cpu_supports("avx2");
    if (avx2)
        stream_copy_avx2(dst, src, n);
    else
        std::memcpy(dst, src, n);
}

// A batch of host copies; `left` counts its unfinished pieces.
struct CopyBatch {
    std::atomic<int64_t> left{0};
};

// Persistent host-copy workers.  submit() splits a range into 1 MiB pieces and
// queues them; wait() blocks until a batch is done, running queued pieces
// itself meanwhile (so a single-core host still makes progress).
class CopyPool {
  public:
    static CopyPool &get() {
        static CopyPool pool;
        return pool;
    }

    void submit(CopyBatch *b, void *dst, const void *src, size_t bytes) {
        if (!bytes) return;
        const int64_t pieces = (int64_t)((bytes + COPY_PIECE - 1) / COPY_PIECE);
        b->left.fetch_add(pieces, std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> g(mu_);
            for (int64_t i = 0; i < pieces; ++i) {
                const size_t off = (size_t)i * COPY_PIECE;
                q_.push_back({static_cast<char *>(dst) + off, static_cast<const char *>(src) + off,
                              std::min(COPY_PIECE, bytes - off), b});
            }
        }
        work_cv_.notify_all();
    }

    void wait(CopyBatch *b) {
        while (b->left.load(std::memory_order_acquire) > 0) {
            Piece p;
            if (pop(&p, /*block=*/false)) {
                run(p);
                continue;
            }
            std::unique_lock<std::mutex> lk(mu_);
            done_cv_.wait(lk, [&] { return b->left.load(std::memory_order_acquire) <= 0 || !q_.empty(); });
        }
    }

    ~CopyPool() {
        {
            std::lock_guard<std::mutex> g(mu_);
            stop_ = true;
        }
        work_cv_.notify_all();
        for (auto &t : threads_) t.join();
    }

  private:
    struct Piece {
        char *dst;
        const char *src;
        size_t bytes;
        CopyBatch *batch;
    };

    CopyPool() {
        unsigned hw = std::thread::hardware_concurrency();
        int n = (int)std::min<unsigned>(hw > 1 ? hw - 1 : 1, 15u);
        for (int i = 0; i < n; ++i) threads_.emplace_back([this] { worker(); });
    }

    bool pop(Piece *p, bool block) {
        std::unique_lock<std::mutex> lk(mu_);
        if (block) work_cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
        if (q_.empty()) return false;
        *p = q_.front();
        q_.pop_front();
        return true;
    }

    void run(const Piece &p) {
        host_copy(p.dst, p.src, p.bytes);
        if (p.batch->left.fetch_sub(1, std::memory_order_acq_rel) == 1) {
            std::lock_guard<std::mutex> g(mu_);  // pairs with the predicate check in wait()
            done_cv_.notify_all();
        }
    }

    void worker() {
        for (;;) {
            Piece p;
            if (!pop(&p, /*block=*/true)) {
                std::lock_guard<std::mutex> g(mu_);
                if (stop_) return;
                continue;
            }
            run(p);
        }
    }

    std::mutex mu_;
    std::condition_variable work_cv_, done_cv_;
    std::deque<Piece> q_;
    std::vector<std::thread> threads_;
    bool stop_ = false;
};

// 1 if [p, p+bytes) is page-locked host memory (registered or cudaHostAlloc'd):
// both ends are checked, so a partially registered range counts as pageable.
inline bool is_pinned(const void *p, size_t bytes) {
    if (!p) return false;
    auto one = [](const void *q) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, q) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    };
    return one(p) && (bytes <= 1 || one(static_cast<const char *>(p) + bytes - 1));
}

// Per-device streams, events and pinned bounce buffers of the pipeline.  `mu`
// serialises whole pipeline calls on one device (the streams, events and
// bounce slots are shared): concurrent callers queue instead of interleaving.
struct Pipe {
    std::mutex mu;
    bool ready = false;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, end_d2h = nullptr;
    cudaEvent_t h2d_done[NSLOT], comp_done[NSLOT], d2h_done[NSLOT];
    char *bounce_in[NSLOT] = {}, *bounce_out[NSLOT] = {};
    size_t bounce_in_bytes = 0, bounce_out_bytes = 0;

    cudaError_t init() {
        if (ready) return cudaSuccess;
        cudaError_t e;
        if ((e = cudaStreamCreateWithFlags(&h2d, cudaStreamNonBlocking)) != cudaSuccess) return e;
        if ((e = cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking)) != cudaSuccess) return e;
        cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&end_d2h, cudaEventDisableTiming);
        for (int i = 0; i < NSLOT; ++i) {
            cudaEventCreateWithFlags(&h2d_done[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&comp_done[i], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&d2h_done[i], cudaEventDisableTiming);
        }
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        ready = true;
        return cudaSuccess;
    }

    // grow the bounce ring to at least in_bytes / out_bytes per slot
    cudaError_t bounce(size_t in_bytes, size_t out_bytes) {
        cudaError_t e;
        if (in_bytes > bounce_in_bytes) {
            for (auto &b : bounce_in) {
                if (b) cudaFreeHost(b);
                b = nullptr;
            }
            for (auto &b : bounce_in)
                if ((e = cudaHostAlloc((void **)&b, in_bytes, cudaHostAllocPortable)) != cudaSuccess) {
                    bounce_in_bytes = 0;
                    return e;
                }
            bounce_in_bytes = in_bytes;
        }
        if (out_bytes > bounce_out_bytes) {
            for (auto &b : bounce_out) {
                if (b) cudaFreeHost(b);
                b = nullptr;
            }
            for (auto &b : bounce_out)
                if ((e = cudaHostAlloc((void **)&b, out_bytes, cudaHostAllocPortable)) != cudaSuccess) {
                    bounce_out_bytes = 0;
                    return e;
                }
            bounce_out_bytes = out_bytes;
        }
        return cudaSuccess;
    }
};

inline int pipe_for_current_device(Pipe **out) {
    static Pipe pipes[64];
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return -1;
    *out = &pipes[dev];
    return 0;
}

// One chunk of the pipeline: byte ranges in the host buffers.
struct Chunk {
    size_t in_off, in_bytes, out_off, out_bytes;
};

// Runs the pipeline over `nchunks` chunks.  chunk_of(k) -> Chunk; launch(k, din,
// dout) enqueues chunk k's compute on `comp` (returns a PS_* code).  The caller
// holds pipe.mu.  On return everything is complete (comp synchronised).
// Returns a cudaError_t-style code through `cuda_err` or the launch's PS code.
template <class ChunkOf, class Launch>
int run(Pipe &P, const char *in_host, char *out_host, int64_t nchunks, size_t in_slot_bytes,
        size_t out_slot_bytes, char *dev_in, char *dev_out, size_t dev_in_slot, size_t dev_out_slot,
        cudaStream_t comp, ChunkOf chunk_of, Launch launch, cudaError_t *cuda_err) {
    *cuda_err = cudaSuccess;
    const Chunk first = chunk_of(0);
    (void)first;
    size_t in_total = 0, out_total = 0;
    for (int64_t k = 0; k < nchunks; ++k) {
        const Chunk c = chunk_of(k);
        in_total = std::max(in_total, c.in_off + c.in_bytes);
        out_total = std::max(out_total, c.out_off + c.out_bytes);
    }
    const bool stage_in = !is_pinned(in_host, in_total);
    const bool stage_out = !is_pinned(out_host, out_total);
    cudaError_t e;
    if ((stage_in || stage_out) &&
        (e = P.bounce(stage_in ? in_slot_bytes : 0, stage_out ? out_slot_bytes : 0)) != cudaSuccess) {
        *cuda_err = e;
        return -1;
    }
    CopyPool &pool = CopyPool::get();
    CopyBatch in_b[NSLOT], out_b[NSLOT];
    auto wait_all = [&] {
        for (auto &b : in_b) pool.wait(&b);
        for (auto &b : out_b) pool.wait(&b);
    };
    auto fail = [&](cudaError_t err) {
        wait_all();
        cudaStreamSynchronize(P.h2d);
        cudaStreamSynchronize(P.d2h);
        cudaStreamSynchronize(comp);
        *cuda_err = err;
        return -1;
    };

    // helper streams start after everything already queued on the caller stream
    if ((e = cudaEventRecord(P.start, comp)) != cudaSuccess) return fail(e);
    cudaStreamWaitEvent(P.h2d, P.start, 0);
    cudaStreamWaitEvent(P.d2h, P.start, 0);

    auto fill = [&](int64_t k) {  // pageable input chunk k -> its bounce slot
        const Chunk c = chunk_of(k);
        pool.submit(&in_b[k % NSLOT], P.bounce_in[k % NSLOT], in_host + c.in_off, c.in_bytes);
    };
    auto drain = [&](int64_t j) -> cudaError_t {  // bounce slot of chunk j -> pageable output
        cudaError_t err = cudaEventSynchronize(P.d2h_done[j % NSLOT]);
        if (err != cudaSuccess) return err;
        const Chunk c = chunk_of(j);
        pool.submit(&out_b[j % NSLOT], out_host + c.out_off, P.bounce_out[j % NSLOT], c.out_bytes);
        return cudaSuccess;
    };

    if (stage_in) fill(0);
    for (int64_t k = 0; k < nchunks; ++k) {
        const int slot = (int)(k % NSLOT);
        const Chunk c = chunk_of(k);
        char *din = dev_in + slot * dev_in_slot;
        char *dout = dev_out + slot * dev_out_slot;
        if (stage_in) pool.wait(&in_b[slot]);
        if (k >= NSLOT) cudaStreamWaitEvent(P.h2d, P.d2h_done[slot], 0);  // device slot free
        e = cudaMemcpyAsync(din, stage_in ? P.bounce_in[slot] : in_host + c.in_off, c.in_bytes,
                            cudaMemcpyHostToDevice, P.h2d);
        if (e != cudaSuccess) return fail(e);
        cudaEventRecord(P.h2d_done[slot], P.h2d);
        // next input chunk into its bounce slot once the H2D that last read it is done
        if (stage_in && k + 1 < nchunks) {
            if (k + 1 >= NSLOT && (e = cudaEventSynchronize(P.h2d_done[(k + 1) % NSLOT])) != cudaSuccess)
                return fail(e);
            fill(k + 1);
        }
        cudaStreamWaitEvent(comp, P.h2d_done[slot], 0);
        int rc = launch(k, din, dout);
        if (rc) {
            fail(cudaSuccess);
            return rc;
        }
        cudaEventRecord(P.comp_done[slot], comp);
        cudaStreamWaitEvent(P.d2h, P.comp_done[slot], 0);
        if (stage_out) pool.wait(&out_b[slot]);  // chunk k-NSLOT drained from this bounce slot
        e = cudaMemcpyAsync(stage_out ? P.bounce_out[slot] : out_host + c.out_off, dout, c.out_bytes,
                            cudaMemcpyDeviceToHost, P.d2h);
        if (e != cudaSuccess) return fail(e);
        cudaEventRecord(P.d2h_done[slot], P.d2h);
        if (stage_out && k >= NSLOT - 1 && (e = drain(k - (NSLOT - 1))) != cudaSuccess) return fail(e);
    }
    if (stage_out)
        for (int64_t j = std::max<int64_t>(0, nchunks - (NSLOT - 1)); j < nchunks; ++j)
            if ((e = drain(j)) != cudaSuccess) return fail(e);
    // the caller stream owns the device workspace again only after the last D2H
    cudaEventRecord(P.end_d2h, P.d2h);
    cudaStreamWaitEvent(comp, P.end_d2h, 0);
    e = cudaStreamSynchronize(comp);
    wait_all();
    if (e != cudaSuccess) {
        *cuda_err = e;
        return -1;
    }
    return 0;
}

}  // namespace host
}  // namespace ps
