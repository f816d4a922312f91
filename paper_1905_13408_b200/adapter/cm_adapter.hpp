// Shared state of the drop-in adapters (regularizer_b200.cpp, params_b200.cpp,
// fourier_b200.cpp): per-thread solver contexts over include/cm_api.h, the
// status -> exception mapping (errors.hpp:7-30), and what is resident on the
// device so that em_refine's M-step block (refine.cpp:174-183, 237-250)
//
//     scales = scale_data(acc);  ...;  x = m_step(acc, x, x, reg);  V = fft3_centered(x);
//
// moves the accumulator to the device once and the result's spectrum comes
// from the resident result instead of a host FFT.
//
// Identity of "the same accumulator / the same volume": the same buffers,
// side and flag, and equal sampled checksums (4096 strided values). em_refine
// hands the very same unmodified objects from one call to the next; a caller
// that rewrites the arrays between calls while keeping every sampled value
// would be missed (documented in INTEGRATION.md).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <utility>

#include "cm_api.h"
#include "cryomap/backproject.hpp"
#include "cryomap/errors.hpp"
#include "cryomap/volume.hpp"

namespace cryomap {
namespace cm_adapter {

[[noreturn]] inline void rethrow(int rc) {
    const std::string msg = cm_last_error();
    switch (rc) {
        case CM_ERR_INVALID_ARGUMENT:
        case CM_ERR_UNSUPPORTED: throw InvalidArgument(msg);
        case CM_ERR_GRID_MISMATCH: throw GridMismatch(msg);
        case CM_ERR_NON_HERMITIAN: throw NonHermitianAccumulator(msg);
        case CM_ERR_STEP_DIVERGED: throw StepDiverged(msg);
        case CM_ERR_NON_POSITIVE_SCALE: throw NonPositiveScale(msg);
        case CM_ERR_NON_HERMITIAN_INPUT: throw NonHermitianInput(msg);
        default: throw Error("cm (B200 solver): " + msg);
    }
}

inline void check(int rc) {
    if (rc != CM_OK) rethrow(rc);
}

// CM_PRECISION=64 (default: the reference's fp64 tests pass unchanged) or 32
inline int precision() {
    const char* p = std::getenv("CM_PRECISION");
    return (p && std::atoi(p) == 32) ? 32 : 64;
}

// the devices a context drives: CM_DEVICES="0,1,2,3" (default "0"); more than one
// device selects the z-slab solver (needs CM_PRECISION=32, sides n % 128 == 0)
inline int devices(int* out, int cap) {
    const char* e = std::getenv("CM_DEVICES");
    int n = 0;
    if (e)
        for (const char* q = e; *q && n < cap;) {
            char* end = nullptr;
            const long v = std::strtol(q, &end, 10);
            if (end == q) break;
            out[n++] = (int)v;
            q = (*end == ',') ? end + 1 : end;
        }
    if (n == 0) out[n++] = 0;
    return n;
}

// sampled checksum of a buffer of doubles (4096 strided values + the length)
inline uint64_t sample_sum(const double* p, size_t count) {
    uint64_t h = 1469598103934665603ull ^ count;
    if (!p || count == 0) return h;
    const size_t step = count > 4096 ? count / 4096 : 1;
    for (size_t i = 0; i < count; i += step) {
        uint64_t b;
        std::memcpy(&b, p + i, 8);
        h = (h ^ b) * 1099511628211ull;
    }
    uint64_t b;
    std::memcpy(&b, p + count - 1, 8);
    return (h ^ b) * 1099511628211ull;
}

struct AccId {
    const void* w = nullptr;
    const void* y = nullptr;
    int n = 0;
    bool fin = false;
    uint64_t sum = 0;
    bool operator==(const AccId& o) const {
        return w == o.w && y == o.y && n == o.n && fin == o.fin && sum == o.sum;
    }
};
inline AccId acc_id(const AccumulatorPair& a) {
    AccId id;
    id.w = a.weight.data();
    id.y = a.numerator.data();
    id.n = a.side_n;
    id.fin = a.finalized;
    id.sum = sample_sum(a.weight.data(), a.weight.size()) ^
             (sample_sum(reinterpret_cast<const double*>(a.numerator.data()), 2 * a.numerator.size()) << 1);
    return id;
}

struct CtxDel {
    void operator()(cm_ctx* c) const { cm_ctx_destroy(c); }
};

struct Slot {
    std::unique_ptr<cm_ctx, CtxDel> ctx;
    bool multi = false;                   // ctx spans several GPUs (z-slab solver)
    std::unique_ptr<cm_ctx, CtxDel> aux;  // multi: one-GPU context for the transforms
    AccId acc;                         // accumulator resident on the device
    bool acc_valid = false;
    const double* result = nullptr;    // host buffer m_step returned, and its checksum
    size_t result_len = 0;
    uint64_t result_sum = 0;
};

inline Slot& slot(int n) {
    thread_local std::map<std::pair<int, int>, Slot> cache;
    const auto key = std::make_pair(n, precision());
    auto it = cache.find(key);
    if (it == cache.end()) {
        require_even_side(n);  // volume.hpp:94-97
        int dev[16];
        const int nd = devices(dev, 16);
        cm_ctx* c = nullptr;
        check(cm_ctx_create(n, dev, nd, key.second, &c));
        it = cache.emplace(key, Slot{}).first;
        it->second.ctx.reset(c);
        it->second.multi = nd > 1;
    }
    return it->second;
}

inline cm_ctx* context(int n) { return slot(n).ctx.get(); }

// the context that runs whole-volume transforms (fft3_centered): the solver's
// own, or for a multi-GPU solver a one-GPU context on its first device
inline cm_ctx* transform_context(Slot& s, int n) {
    if (!s.multi) return s.ctx.get();
    if (!s.aux) {
        int dev[16];
        devices(dev, 16);
        cm_ctx* c = nullptr;
        check(cm_ctx_create(n, dev, 1, precision(), &c));
        s.aux.reset(c);
    }
    return s.aux.get();
}

// make `acc` the resident accumulator (no upload when it already is)
inline void upload_acc(Slot& s, const AccumulatorPair& acc) {
    const AccId id = acc_id(acc);
    if (s.acc_valid && s.acc == id) return;
    s.acc_valid = false;
    check(cm_set_accumulator(s.ctx.get(), acc.weight.data(),
                             reinterpret_cast<const double*>(acc.numerator.data()),
                             acc.finalized ? 1 : 0));
    s.acc = id;
    s.acc_valid = true;
}

// a one-GPU context holding `acc` for the component entry points (data_gradient,
// penalized_objective): the solver's own, or the transform context of a
// multi-GPU solver
inline cm_ctx* component_context(const AccumulatorPair& acc) {
    Slot& s = slot(acc.side_n);
    if (!s.multi) {
        upload_acc(s, acc);
        return s.ctx.get();
    }
    cm_ctx* c = transform_context(s, acc.side_n);
    check(cm_set_accumulator(c, acc.weight.data(), reinterpret_cast<const double*>(acc.numerator.data()),
                             acc.finalized ? 1 : 0));
    return c;
}

inline void note_result(Slot& s, const Volume3D& out) {
    s.result = out.data.data();
    s.result_len = out.data.size();
    s.result_sum = sample_sum(out.data.data(), out.data.size());
}

inline bool is_result(const Slot& s, const Volume3D& v) {
    return s.result && !s.multi && v.data.data() == s.result && v.data.size() == s.result_len &&
           sample_sum(v.data.data(), v.data.size()) == s.result_sum;
}

} // namespace cm_adapter
} // namespace cryomap
