// One translation unit per side length (built in parallel by build.py).
#ifdef CM_STUB
#include <string>
namespace cm { struct ImplBase; struct DistBase; }
#else
#include "dist.cuh"
#include "impl.cuh"
#endif

#ifndef CM_N
#error "CM_N must be defined"
#endif

#define CM_CAT2(a, b) a##b
#define CM_CAT(a, b) CM_CAT2(a, b)

namespace cm {
ImplBase* CM_CAT(make_impl_, CM_N)(int precision) {
#ifdef CM_STUB
    (void)precision;
    return nullptr; // side compiled out of a development build
#else
    if (precision == 64) return new Impl<double, CM_N>();
    return new Impl<float, CM_N>();
#endif
}

// z-slab solver: fp32 sides with the 128-wide stencil tiles
DistBase* CM_CAT(make_dist_, CM_N)() {
#if !defined(CM_STUB) && (CM_N % 128 == 0)
    return new DistImpl<CM_N>();
#else
    return nullptr;
#endif
}
} // namespace cm
