// Host <-> device transfers of the drop-in's PAGEABLE buffers.
//
// The reference API hands the solver plain std::vector storage
// (regularizer.hpp:98-100: AccumulatorPair, Volume3D by const&; the result
// returned by value), i.e. pageable memory. cudaMemcpyAsync from pageable
// memory is synchronous and staged by the driver through small bounce
// buffers. HostXfer instead streams such buffers through a ring of pinned
// 64 MiB chunks: the host copy of chunk i+1 (split over a few threads) runs
// while the DMA of chunk i is in flight on the context's stream, so the
// transfer runs at the PCIe rate rather than memcpy + DMA in series.
// Pinned (page-locked or cudaHostRegister'ed) host pointers go straight to
// cudaMemcpyAsync.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cm_api.h"

namespace cm {

int fail(int code, const std::string& msg);

// A persistent pool of copy threads (thread creation per 64 MiB chunk cost
// ~20 us x threads x chunks: a few percent of a 5 GB transfer). A job is a
// destination range [0, bytes) filled from a list of source segments (one
// segment: a plain memcpy); worker t of nt copies [t part, (t+1) part).
struct CopySeg {
    const void* src;
    size_t bytes;
};

inline void copy_segments(unsigned char* dst, const CopySeg* segs, size_t nseg, size_t lo, size_t hi) {
    size_t off = 0;
    for (size_t s = 0; s < nseg && off < hi; ++s) {
        const size_t end = off + segs[s].bytes;
        if (end > lo) {
            const size_t a = std::max(off, lo), b = std::min(end, hi);
            std::memcpy(dst + a, (const unsigned char*)segs[s].src + (a - off), b - a);
        }
        off = end;
    }
}

struct CopyPool {
    std::vector<std::thread> th;
    std::mutex m;
    std::condition_variable cv, done_cv;
    unsigned char* dst = nullptr;
    const CopySeg* segs = nullptr;
    size_t nseg = 0, part = 0, bytes = 0;
    int gen = 0, pending = 0;
    bool quit = false;
    explicit CopyPool(int n) {
        for (int t = 1; t < n; ++t)  // the caller is worker 0
            th.emplace_back([this, t] {
                int seen = 0;
                for (;;) {
                    std::unique_lock<std::mutex> lk(m);
                    cv.wait(lk, [&] { return quit || gen != seen; });
                    if (quit) return;
                    seen = gen;
                    const size_t lo = std::min(part * t, bytes), hi = std::min(lo + part, bytes);
                    unsigned char* d = dst;
                    const CopySeg* sg = segs;
                    const size_t ns = nseg;
                    lk.unlock();
                    if (hi > lo) copy_segments(d, sg, ns, lo, hi);
                    lk.lock();
                    if (--pending == 0) done_cv.notify_one();
                }
            });
    }
    ~CopyPool() {
        {
            std::lock_guard<std::mutex> lk(m);
            quit = true;
        }
        cv.notify_all();
        for (auto& t : th) t.join();
    }
    int size() const { return (int)th.size() + 1; }
    void copy(void* d, const CopySeg* sg, size_t ns, size_t n) {
        const int nt = size();
        const size_t prt = (n / nt + 4095) & ~size_t(4095);
        {
            std::lock_guard<std::mutex> lk(m);
            dst = (unsigned char*)d;
            segs = sg;
            nseg = ns;
            part = prt;
            bytes = n;
            pending = nt - 1;
            ++gen;
        }
        cv.notify_all();
        copy_segments((unsigned char*)d, sg, ns, 0, std::min(prt, n));
        std::unique_lock<std::mutex> lk(m);
        done_cv.wait(lk, [&] { return pending == 0; });
    }
    void copy(void* d, const void* sp, size_t n) {
        const CopySeg one{sp, n};
        copy(d, &one, 1, n);
    }
};

struct HostXfer {
    static constexpr size_t kChunk = size_t(64) << 20;
    static constexpr int kBufs = 3;
    unsigned char* buf[kBufs] = {};
    cudaEvent_t done[kBufs] = {};
    // host copy threads: CM_XFER_THREADS, default the hardware threads (<= 16);
    // measured on the B200 box (16 threads): 4 -> 25.7, 8 -> 34.3, 16 -> 37.4 GB/s
    // for the 5.4 GB of one 512^3 cm_m_step
    int threads = []() {
        if (const char* e = std::getenv("CM_XFER_THREADS")) return std::max(1, std::atoi(e));
        return (int)std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    }();
    std::unique_ptr<CopyPool> pool;

    ~HostXfer() {
        pool.reset();
        for (int q = 0; q < kBufs; ++q) {
            if (buf[q]) cudaFreeHost(buf[q]);
            if (done[q]) cudaEventDestroy(done[q]);
        }
    }
    int ensure() {
        for (int q = 0; q < kBufs; ++q) {
            if (!buf[q] && cudaHostAlloc((void**)&buf[q], kChunk, cudaHostAllocDefault) != cudaSuccess)
                return fail(CM_ERR_CUDA, "pinned staging allocation failed");
            if (!done[q] && cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming) != cudaSuccess)
                return fail(CM_ERR_CUDA, "staging event creation failed");
        }
        if (!pool && threads > 1) pool.reset(new CopyPool(threads));
        return CM_OK;
    }
    static bool pinned(const void* p) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return false;
        }
        return a.type == cudaMemoryTypeHost;
    }
    // memcpy split over the pool (host-side bandwidth of one core is well below
    // the PCIe rate)
    void pcopy(void* dst, const void* src, size_t bytes) const {
        if (!pool || bytes < (size_t(8) << 20)) {
            std::memcpy(dst, src, bytes);
            return;
        }
        pool->copy(dst, src, bytes);
    }

    void pcopy_segs(void* dst, const CopySeg* segs, size_t nseg, size_t bytes) const {
        if (!pool || bytes < (size_t(8) << 20)) {
            copy_segments((unsigned char*)dst, segs, nseg, 0, bytes);
            return;
        }
        pool->copy(dst, segs, nseg, bytes);
    }

    // gather: the segments, concatenated in order, land contiguously at dev
    // (pageable sources packed into the pinned ring by the copy pool). Same
    // completion semantics as h2d.
    int h2d_segments(void* dev, const std::vector<CopySeg>& segs, cudaStream_t st) {
        if (segs.empty()) return CM_OK;
        if (pinned(segs[0].src)) {
            size_t off = 0;
            for (const CopySeg& g : segs) {
                if (cudaMemcpyAsync((unsigned char*)dev + off, g.src, g.bytes, cudaMemcpyHostToDevice, st) !=
                    cudaSuccess)
                    return fail(CM_ERR_CUDA, "host-to-device copy failed");
                off += g.bytes;
            }
            return CM_OK;
        }
        if (int rc = ensure()) return rc;
        size_t s = 0, soff = 0, doff = 0;  // next source byte: segment s, offset soff
        std::vector<CopySeg> cur;
        for (int i = 0; s < segs.size(); ++i) {
            const int b = i % kBufs;
            // the chunk's segment list (the first and last may be partial)
            cur.clear();
            size_t len = 0;
            while (s < segs.size() && len < kChunk) {
                const size_t take = std::min(segs[s].bytes - soff, kChunk - len);
                cur.push_back({(const unsigned char*)segs[s].src + soff, take});
                len += take;
                soff += take;
                if (soff == segs[s].bytes) {
                    ++s;
                    soff = 0;
                }
            }
            if (cudaEventSynchronize(done[b]) != cudaSuccess) return fail(CM_ERR_CUDA, "staging wait failed");
            pcopy_segs(buf[b], cur.data(), cur.size(), len);
            if (cudaMemcpyAsync((unsigned char*)dev + doff, buf[b], len, cudaMemcpyHostToDevice, st) !=
                    cudaSuccess ||
                cudaEventRecord(done[b], st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "host-to-device copy failed");
            doff += len;
        }
        return CM_OK;
    }

    // stream-ordered on return for pinned sources; for pageable sources the
    // host buffer may be reused on return (the last chunk is in flight from the
    // pinned ring, which the next call waits for)
    int h2d(void* dev, const void* host, size_t bytes, cudaStream_t st) {
        if (bytes == 0) return CM_OK;
        if (pinned(host)) {
            if (cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "host-to-device copy failed");
            return CM_OK;
        }
        if (int rc = ensure()) return rc;
        size_t off = 0;
        for (int i = 0; off < bytes; ++i, off += kChunk) {
            const int b = i % kBufs;
            const size_t len = std::min(kChunk, bytes - off);
            if (cudaEventSynchronize(done[b]) != cudaSuccess)
                return fail(CM_ERR_CUDA, "staging wait failed");
            pcopy(buf[b], (const unsigned char*)host + off, len);
            if (cudaMemcpyAsync((unsigned char*)dev + off, buf[b], len, cudaMemcpyHostToDevice, st) !=
                    cudaSuccess ||
                cudaEventRecord(done[b], st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "host-to-device copy failed");
        }
        return CM_OK;
    }

    // synchronous: the host buffer holds the data on return
    int d2h(void* host, const void* dev, size_t bytes, cudaStream_t st) {
        if (bytes == 0) return CM_OK;
        if (pinned(host)) {
            if (cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "device-to-host copy failed");
            return CM_OK;
        }
        if (int rc = ensure()) return rc;
        const size_t nchunk = (bytes + kChunk - 1) / kChunk;
        auto issue = [&](size_t i) -> int {
            const int b = (int)(i % kBufs);
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            if (cudaMemcpyAsync(buf[b], (const unsigned char*)dev + off, len, cudaMemcpyDeviceToHost,
                                st) != cudaSuccess ||
                cudaEventRecord(done[b], st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "device-to-host copy failed");
            return CM_OK;
        };
        // keep kBufs-1 chunks in flight ahead of the host copy
        for (size_t i = 0; i < std::min(nchunk, (size_t)kBufs - 1); ++i)
            if (int rc = issue(i)) return rc;
        for (size_t i = 0; i < nchunk; ++i) {
            const int b = (int)(i % kBufs);
            if (cudaEventSynchronize(done[b]) != cudaSuccess)
                return fail(CM_ERR_CUDA, "device-to-host copy failed");
            if (i + kBufs - 1 < nchunk)
                if (int rc = issue(i + kBufs - 1)) return rc;
            const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
            pcopy((unsigned char*)host + off, buf[b], len);
        }
        return CM_OK;
    }
};

} // namespace cm
