// Collectives of the z-slab distributed solver.
//
// Two backends behind one interface, both stream-ordered:
//   * NcclComm — one rank per process/GPU, NCCL loaded at run time (dlopen of
//     libnccl.so.2, the copy torch ships), grouped ncclSend/ncclRecv for the
//     all-to-all transposes and the halo planes, ncclAllGather, ncclAllReduce;
//   * EmuComm  — P virtual ranks inside one process on one GPU (correctness
//     tests of the decomposition): the same exchanges as device-to-device copies.
// A "group" call gets the buffers of all virtual ranks this process hosts
// (P for EmuComm, 1 for NcclComm).
#pragma once

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstdlib>

#include <string>
#include <vector>

namespace cm {

// ---- minimal NCCL ABI (nccl.h types; resolved with dlsym) -------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef enum { ncclSuccess = 0 } ncclResult_t;
typedef enum { ncclChar = 0, ncclFloat64 = 8 } ncclDataType_t;
typedef enum { ncclSum = 0 } ncclRedOp_t;

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;

    bool load(std::string* err) {
        if (h) return true;
        const char* env = std::getenv("CM_NCCL_LIBRARY");
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* n : names)
            if (n && (h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            *err = "libnccl.so.2 not found (set CM_NCCL_LIBRARY)";
            return false;
        }
#define CM_SYM(f) f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f)); if (!f) { *err = "missing nccl" #f; return false; }
        CM_SYM(GetUniqueId) CM_SYM(CommInitRank) CM_SYM(CommDestroy) CM_SYM(Send) CM_SYM(Recv)
        CM_SYM(AllGather) CM_SYM(AllReduce) CM_SYM(GroupStart) CM_SYM(GroupEnd) CM_SYM(GetErrorString)
#undef CM_SYM
        return true;
    }
};

inline NcclApi& nccl_api() {
    static NcclApi api;
    return api;
}

struct Comm {
    int P = 1;        // total ranks
    int nv = 1;       // virtual ranks hosted by this process
    int rank0 = 0;    // global rank of virtual rank 0
    virtual ~Comm() = default;
    // all-to-all: send[v] holds P chunks of `bytes` (chunk s -> rank s); recv[v]
    // receives chunk r from rank r at offset r*bytes
    virtual int all_to_all(const std::vector<void*>& send, const std::vector<void*>& recv,
                           size_t bytes, cudaStream_t s) = 0;
    // halo: lo[v]/hi[v] are the first/last interior planes, glo[v]/ghi[v] the ghost
    // planes below/above; rank r's hi -> rank r+1's glo, r's lo -> r-1's ghi
    virtual int halo(const std::vector<void*>& lo, const std::vector<void*>& hi,
                     const std::vector<void*>& glo, const std::vector<void*>& ghi, size_t bytes,
                     cudaStream_t s) = 0;
    virtual int all_gather(const std::vector<void*>& mine, const std::vector<void*>& all,
                           size_t bytes, cudaStream_t s) = 0;
    // in-place sum of `count` doubles over all ranks
    virtual int all_reduce_sum(const std::vector<double*>& buf, int count, cudaStream_t s) = 0;
};

__global__ static void emu_sum_kernel(double* const* bufs, int nv, int count) {
    const int q = threadIdx.x;
    if (q >= count) return;
    double s = 0.0;
    for (int v = 0; v < nv; ++v) s += bufs[v][q];  // fixed rank order
    for (int v = 0; v < nv; ++v) bufs[v][q] = s;
}

struct EmuComm final : Comm {
    double** dptrs = nullptr;
    explicit EmuComm(int p) {
        P = p;
        nv = p;
        cudaMalloc((void**)&dptrs, sizeof(double*) * p);
    }
    ~EmuComm() override {
        if (dptrs) cudaFree(dptrs);
    }
    int all_to_all(const std::vector<void*>& send, const std::vector<void*>& recv, size_t bytes,
                   cudaStream_t s) override {
        for (int r = 0; r < P; ++r)
            for (int d = 0; d < P; ++d)
                if (cudaMemcpyAsync((char*)recv[d] + (size_t)r * bytes, (char*)send[r] + (size_t)d * bytes,
                                    bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
                    return 1;
        return 0;
    }
    int halo(const std::vector<void*>& lo, const std::vector<void*>& hi,
             const std::vector<void*>& glo, const std::vector<void*>& ghi, size_t bytes,
             cudaStream_t s) override {
        for (int r = 0; r < P; ++r) {
            if (r + 1 < P && cudaMemcpyAsync(glo[r + 1], hi[r], bytes, cudaMemcpyDeviceToDevice, s))
                return 1;
            if (r > 0 && cudaMemcpyAsync(ghi[r - 1], lo[r], bytes, cudaMemcpyDeviceToDevice, s))
                return 1;
        }
        return 0;
    }
    int all_gather(const std::vector<void*>& mine, const std::vector<void*>& all, size_t bytes,
                   cudaStream_t s) override {
        for (int d = 0; d < P; ++d)
            for (int r = 0; r < P; ++r)
                if (cudaMemcpyAsync((char*)all[d] + (size_t)r * bytes, mine[r], bytes,
                                    cudaMemcpyDeviceToDevice, s))
                    return 1;
        return 0;
    }
    int all_reduce_sum(const std::vector<double*>& buf, int count, cudaStream_t s) override {
        if (cudaMemcpyAsync(dptrs, buf.data(), sizeof(double*) * P, cudaMemcpyHostToDevice, s))
            return 1;
        emu_sum_kernel<<<1, 32, 0, s>>>(dptrs, P, count);
        return cudaGetLastError() != cudaSuccess;
    }
};

struct NcclComm final : Comm {
    ncclComm_t comm = nullptr;
    NcclApi* api = nullptr;
    std::string err;
    NcclComm(int p, int rank, const ncclUniqueId& id, int* status) {
        P = p;
        nv = 1;
        rank0 = rank;
        api = &nccl_api();
        *status = (api->load(&err) && api->CommInitRank(&comm, p, id, rank) == ncclSuccess) ? 0 : 1;
    }
    ~NcclComm() override {
        if (comm) api->CommDestroy(comm);
    }
    int all_to_all(const std::vector<void*>& send, const std::vector<void*>& recv, size_t bytes,
                   cudaStream_t s) override {
        int bad = api->GroupStart();
        for (int d = 0; d < P; ++d) {
            bad |= api->Send((char*)send[0] + (size_t)d * bytes, bytes, ncclChar, d, comm, s);
            bad |= api->Recv((char*)recv[0] + (size_t)d * bytes, bytes, ncclChar, d, comm, s);
        }
        bad |= api->GroupEnd();
        return bad;
    }
    int halo(const std::vector<void*>& lo, const std::vector<void*>& hi,
             const std::vector<void*>& glo, const std::vector<void*>& ghi, size_t bytes,
             cudaStream_t s) override {
        int bad = api->GroupStart();
        if (rank0 + 1 < P) {
            bad |= api->Send(hi[0], bytes, ncclChar, rank0 + 1, comm, s);
            bad |= api->Recv(ghi[0], bytes, ncclChar, rank0 + 1, comm, s);
        }
        if (rank0 > 0) {
            bad |= api->Send(lo[0], bytes, ncclChar, rank0 - 1, comm, s);
            bad |= api->Recv(glo[0], bytes, ncclChar, rank0 - 1, comm, s);
        }
        bad |= api->GroupEnd();
        return bad;
    }
    int all_gather(const std::vector<void*>& mine, const std::vector<void*>& all, size_t bytes,
                   cudaStream_t s) override {
        return api->AllGather(mine[0], all[0], bytes, ncclChar, comm, s);
    }
    int all_reduce_sum(const std::vector<double*>& buf, int count, cudaStream_t s) override {
        return api->AllReduce(buf[0], buf[0], (size_t)count, ncclFloat64, ncclSum, comm, s);
    }
};

} // namespace cm
