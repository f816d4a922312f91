// MRC volume I/O straight to and from the resident device volumes (host side of
// cm_set_volumes_mrc / cm_write_volume_mrc).
//
// Format and checks follow the reference reader / writer
// (/root/reference/proj/src/mrc.cpp): a 1024-byte little-endian header, then a
// mode-2 float32 payload, x fastest -- exactly the device layout of an fp32
// volume. So no fp64 detour: the payload streams from the file through two
// pinned chunks into HBM (the read of chunk c+1 overlaps the copy of chunk c),
// and back out the same way. The header statistics are the writer's
// sequential fp64 sums (mrc.cpp:57-74), accumulated chunk by chunk in file
// order, so the bytes match write_mrc(path, Volume3D) exactly.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <string>
#include <thread>

#include "../../include/cm_api.h"

namespace cm {

int fail(int code, const std::string& msg);

static_assert(__BYTE_ORDER__ == __ORDER_LITTLE_ENDIAN__,
              "MRC payloads are little-endian; this host path copies them verbatim");

constexpr size_t kMrcHeader = 1024;
constexpr size_t kMrcChunk = size_t(16) << 20;  // floats per pinned chunk (64 MiB)

inline int32_t mrc_i32(const unsigned char* h, size_t off) {
    int32_t v;
    std::memcpy(&v, h + off, 4);
    return v;
}
inline float mrc_f32(const unsigned char* h, size_t off) {
    float v;
    std::memcpy(&v, h + off, 4);
    return v;
}
inline void mrc_put(unsigned char* h, size_t off, int32_t v) { std::memcpy(h + off, &v, 4); }
inline void mrc_putf(unsigned char* h, size_t off, float v) { std::memcpy(h + off, &v, 4); }

// Two pinned chunks and their copy-done events, owned by a context on first use.
struct MrcRing {
    float* buf[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    ~MrcRing() {
        for (int q = 0; q < 2; ++q) {
            if (buf[q]) cudaFreeHost(buf[q]);
            if (done[q]) cudaEventDestroy(done[q]);
        }
    }
    int ensure() {
        for (int q = 0; q < 2; ++q) {
            if (!buf[q] && cudaHostAlloc((void**)&buf[q], kMrcChunk * 4, cudaHostAllocDefault) !=
                               cudaSuccess)
                return fail(CM_ERR_CUDA, "mrc: pinned staging allocation failed");
            if (!done[q] && cudaEventCreateWithFlags(&done[q], cudaEventDisableTiming) != cudaSuccess)
                return fail(CM_ERR_CUDA, "mrc: event creation failed");
        }
        return CM_OK;
    }
};

struct MrcFile {
    FILE* f = nullptr;
    ~MrcFile() {
        if (f) std::fclose(f);
    }
};

// read_mrc's checks (mrc.cpp:156-199) followed by read_mrc_volume's
// (mrc.cpp:219-224); on success *data_off is the payload offset. `n` is the
// context's side: a readable volume of another side is a grid mismatch.
inline int mrc_open_volume(const char* path, int n, MrcFile& mf, size_t* data_off) {
    const std::string p(path);
    mf.f = std::fopen(path, "rb");
    if (!mf.f) return fail(CM_ERR_IO, "read_mrc: cannot open " + p);
    if (std::fseek(mf.f, 0, SEEK_END) != 0) return fail(CM_ERR_IO, "read_mrc: read failure on " + p);
    const long long size = std::ftell(mf.f);
    if (size < 0 || std::fseek(mf.f, 0, SEEK_SET) != 0)
        return fail(CM_ERR_IO, "read_mrc: read failure on " + p);
    if ((size_t)size < kMrcHeader)
        return fail(CM_ERR_TRUNCATED_FILE, "read_mrc: file shorter than the 1024-byte header");
    unsigned char h[kMrcHeader];
    if (std::fread(h, 1, kMrcHeader, mf.f) != kMrcHeader)
        return fail(CM_ERR_IO, "read_mrc: read failure on " + p);
    if (!(h[208] == 'M' && h[209] == 'A' && h[210] == 'P' && h[211] == ' '))
        return fail(CM_ERR_BAD_MAGIC, "read_mrc: missing \"MAP \" identifier at offset 208");
    const int32_t mode = mrc_i32(h, 12);
    if (mode != 2)
        return fail(CM_ERR_UNSUPPORTED_MODE, "read_mrc: mode " + std::to_string(mode) +
                                                 " (only mode 2 float32 is supported)");
    const int64_t nx = mrc_i32(h, 0), ny = mrc_i32(h, 4), nz = mrc_i32(h, 8);
    if (nx <= 0 || ny <= 0 || nz <= 0 || nx != ny)
        return fail(CM_ERR_INVALID_ARGUMENT, "read_mrc: invalid dimensions");
    const int64_t nsymbt = mrc_i32(h, 92);
    if (nsymbt < 0) return fail(CM_ERR_INVALID_ARGUMENT, "read_mrc: negative extended header size");
    const int64_t nval = nx * ny * nz;
    if (nval > (int64_t)std::numeric_limits<int32_t>::max())
        return fail(CM_ERR_INVALID_ARGUMENT, "read_mrc: payload too large");
    const int64_t need = (int64_t)kMrcHeader + nsymbt + nval * 4;
    if (size < need)
        return fail(CM_ERR_TRUNCATED_FILE, "read_mrc: file shorter than header + payload (" +
                                               std::to_string(size) + " < " +
                                               std::to_string(need) + " bytes)");
    const bool is_volume = mrc_i32(h, 88) == 1 && nz > 1;
    if (is_volume && nz != nx)
        return fail(CM_ERR_INVALID_ARGUMENT, "read_mrc: volume flag set but nz != nx");
    if (!is_volume)
        return fail(CM_ERR_INVALID_ARGUMENT, "read_mrc_volume: " + p + " holds an image stack");
    if (nx != n)
        return fail(CM_ERR_GRID_MISMATCH, "mrc: volume side " + std::to_string(nx) +
                                              " != context side " + std::to_string(n));
    *data_off = kMrcHeader + (size_t)nsymbt;
    return CM_OK;
}

// file payload -> device floats, chunked through the pinned ring on `stream`
inline int mrc_read_payload(MrcFile& mf, size_t data_off, float* dev, size_t L, MrcRing& ring,
                            cudaStream_t stream) {
    if (std::fseek(mf.f, (long)data_off, SEEK_SET) != 0)
        return fail(CM_ERR_IO, "read_mrc: read failure");
    int q = 0;
    for (size_t off = 0; off < L; off += kMrcChunk, q ^= 1) {
        const size_t cnt = L - off < kMrcChunk ? L - off : kMrcChunk;
        if (cudaEventSynchronize(ring.done[q]) != cudaSuccess)
            return fail(CM_ERR_CUDA, "mrc: staging copy failed");
        if (std::fread(ring.buf[q], 4, cnt, mf.f) != cnt)
            return fail(CM_ERR_IO, "read_mrc: read failure");
        if (cudaMemcpyAsync(dev + off, ring.buf[q], cnt * 4, cudaMemcpyHostToDevice, stream) !=
                cudaSuccess ||
            cudaEventRecord(ring.done[q], stream) != cudaSuccess)
            return fail(CM_ERR_CUDA, "mrc: host-to-device copy failed");
    }
    return CM_OK;
}

// device floats -> file (header with the writer's statistics), mrc.cpp:76-144
inline int mrc_write_volume(const char* path, int n, double voxel_size, const float* dev,
                            MrcRing& ring, cudaStream_t stream) {
    const std::string p(path);
    const size_t L = (size_t)n * n * n;
    MrcFile mf;
    mf.f = std::fopen(path, "wb");
    if (!mf.f) return fail(CM_ERR_IO, "write_mrc: cannot open " + p);
    unsigned char h[kMrcHeader];
    std::memset(h, 0, sizeof h);
    if (std::fwrite(h, 1, kMrcHeader, mf.f) != kMrcHeader)
        return fail(CM_ERR_IO, "write_mrc: short write to " + p);
    // D2H of chunk c+1 is in flight while chunk c is summed and written
    double mn = 0.0, mx = 0.0, sum = 0.0, sum2 = 0.0;
    const size_t nchunks = (L + kMrcChunk - 1) / kMrcChunk;
    auto issue = [&](size_t c) -> int {
        const size_t off = c * kMrcChunk, cnt = L - off < kMrcChunk ? L - off : kMrcChunk;
        if (cudaMemcpyAsync(ring.buf[c & 1], dev + off, cnt * 4, cudaMemcpyDeviceToHost, stream) !=
                cudaSuccess ||
            cudaEventRecord(ring.done[c & 1], stream) != cudaSuccess)
            return fail(CM_ERR_CUDA, "mrc: device-to-host copy failed");
        return CM_OK;
    };
    if (nchunks > 0) {
        const int st = issue(0);
        if (st) return st;
    }
    for (size_t c = 0; c < nchunks; ++c) {
        if (c + 1 < nchunks) {
            const int st = issue(c + 1);
            if (st) return st;
        }
        if (cudaEventSynchronize(ring.done[c & 1]) != cudaSuccess)
            return fail(CM_ERR_CUDA, "mrc: device-to-host copy failed");
        const size_t off = c * kMrcChunk, cnt = L - off < kMrcChunk ? L - off : kMrcChunk;
        const float* b = ring.buf[c & 1];
        if (c == 0) mn = mx = b[0];
        // the sequential statistics (a dependent fp64 add chain per sum, so not
        // parallelisable bit-exactly) run beside the file write, one chain per thread
        std::thread t_sum([&, b, cnt] {
            double a = sum;  // register-resident: no false sharing between chains
            for (size_t i = 0; i < cnt; ++i) a += b[i];
            sum = a;
        });
        std::thread t_sum2([&, b, cnt] {
            double a = sum2;
            for (size_t i = 0; i < cnt; ++i) a += double(b[i]) * b[i];
            sum2 = a;
        });
        std::thread t_ext([&, b, cnt] {
            double lo = mn, hi = mx;
            for (size_t i = 0; i < cnt; ++i) {
                const double v = b[i];
                lo = v < lo ? v : lo;  // std::min / std::max order (mrc.cpp:63-64)
                hi = v > hi ? v : hi;
            }
            mn = lo;
            mx = hi;
        });
        const bool wrote = std::fwrite(b, 4, cnt, mf.f) == cnt;
        t_sum.join();
        t_sum2.join();
        t_ext.join();
        if (!wrote) return fail(CM_ERR_IO, "write_mrc: short write to " + p);
    }
    const double mean = sum / (double)L;
    double var = sum2 / (double)L - mean * mean;
    var = var > 0.0 ? var : 0.0;
    mrc_put(h, 0, n);
    mrc_put(h, 4, n);
    mrc_put(h, 8, n);
    mrc_put(h, 12, 2);
    mrc_put(h, 28, n);
    mrc_put(h, 32, n);
    mrc_put(h, 36, n);
    const float cx = float(n * voxel_size);
    const double unit = double(cx) / n;
    mrc_putf(h, 40, cx);
    mrc_putf(h, 44, float(n * unit));
    mrc_putf(h, 48, float(n * unit));
    mrc_putf(h, 52, 90.0f);
    mrc_putf(h, 56, 90.0f);
    mrc_putf(h, 60, 90.0f);
    mrc_put(h, 64, 1);
    mrc_put(h, 68, 2);
    mrc_put(h, 72, 3);
    mrc_putf(h, 76, float(mn));
    mrc_putf(h, 80, float(mx));
    mrc_putf(h, 84, float(mean));
    mrc_put(h, 88, 1);
    mrc_put(h, 92, 0);
    std::memcpy(h + 208, "MAP ", 4);
    h[212] = 0x44;
    h[213] = 0x44;
    mrc_putf(h, 216, float(std::sqrt(var)));
    if (std::fseek(mf.f, 0, SEEK_SET) != 0 || std::fwrite(h, 1, kMrcHeader, mf.f) != kMrcHeader)
        return fail(CM_ERR_IO, "write_mrc: short write to " + p);
    if (std::fclose(mf.f) != 0) {
        mf.f = nullptr;
        return fail(CM_ERR_IO, "write_mrc: short write to " + p);
    }
    mf.f = nullptr;
    return CM_OK;
}

} // namespace cm
