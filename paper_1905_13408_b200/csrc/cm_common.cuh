// Shared device helpers for the B200 M-step solver (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace cm {

// ---- real / complex traits (fp32 product mode, fp64 parity mode) ----------
template <typename R> struct CxT;
template <> struct CxT<float> { using type = float2; };
template <> struct CxT<double> { using type = double2; };
template <typename R> using Cx = typename CxT<R>::type;

template <typename C> __device__ __forceinline__ C cx(decltype(C::x) re, decltype(C::x) im) {
    C c;
    c.x = re;
    c.y = im;
    return c;
}
template <typename C> __device__ __forceinline__ C cadd(C a, C b) { return cx<C>(a.x + b.x, a.y + b.y); }
template <typename C> __device__ __forceinline__ C csub(C a, C b) { return cx<C>(a.x - b.x, a.y - b.y); }
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    return cx<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a * conj(b)
template <typename C> __device__ __forceinline__ C cmulc(C a, C b) {
    return cx<C>(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
}
template <typename C> __device__ __forceinline__ C cconj(C a) { return cx<C>(a.x, -a.y); }
template <typename C, typename R> __device__ __forceinline__ C cscale(C a, R s) {
    return cx<C>(a.x * s, a.y * s);
}
#ifndef CM_FADD2
#define CM_FADD2 1
#endif
#ifndef CM_PACKED_TW
#define CM_PACKED_TW 0
#endif
#if CM_FADD2
// fp32 complex add / sub as packed FADD2 (sm_100a fp32x2 pipe)
__device__ __forceinline__ float2 cadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 csub(float2 a, float2 b) {
    unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a);
    unsigned long long rb = *reinterpret_cast<unsigned long long*>(&b), rd;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
    return *reinterpret_cast<float2*>(&rd);
}
#endif

// Twiddle sources for the FFT engine. Plain: a table of w = exp(-2 pi i q/TWN)
// (conj for the inverse). Packed (fp32): per entry {w, i w} of the direction
// in use, so u * w = FFMA2(u.y, i w, FMUL2(u.x, w)) — two packed instructions.
template <typename C, bool FWD> struct TwPlain {
    const C* tw;
    __device__ __forceinline__ C mul(C u, int q) const {
        const C w = tw[q];
        return FWD ? cmul(u, w) : cmulc(u, w);
    }
};
// Same table, but a radix-R stage reads only w^k and forms w^(rk) by complex
// products (depth <= 6: error ~6 ulp). For the x lines, where the lanes of a
// warp read 16 different k at stride 2r (up to 16-way bank conflicts), this
// trades 14 shared loads per 16 elements for FMA work.
template <typename C, bool FWD> struct TwPow {
    static constexpr bool kPow = true;
    const C* tw;
    __device__ __forceinline__ C get(int q) const {
        const C w = tw[q];
        return FWD ? w : cx<C>(w.x, -w.y);
    }
    __device__ __forceinline__ C mul(C u, int q) const {
        const C w = tw[q];
        return FWD ? cmul(u, w) : cmulc(u, w);
    }
};
template <typename T, typename = void> struct tw_has_pow { static constexpr bool value = false; };
template <typename T> struct tw_has_pow<T, decltype((void)T::kPow, void())> {
    static constexpr bool value = T::kPow;
};

struct TwPacked {
    const float4* tw4;
    __device__ __forceinline__ float2 mul(float2 u, int q) const {
        const float4 w = tw4[q];
        return __ffma2_rn(make_float2(u.y, u.y), make_float2(w.z, w.w),
                          __fmul2_rn(make_float2(u.x, u.x), make_float2(w.x, w.y)));
    }
};

// multiply by -i (fwd=true) or +i
template <bool FWD, typename C> __device__ __forceinline__ C cmul_mi(C a) {
    return FWD ? cx<C>(a.y, -a.x) : cx<C>(-a.y, a.x);
}

// ---- solver device state (one per context, in device memory) --------------
// Written by the per-iteration finalize kernel; read by every kernel of the
// iteration so that a captured CUDA graph can stop early on the device.
struct DevState {
    int iter;          // iterations completed (index of the next iteration)
    int max_iters;     // inner_iters
    int done;          // 1: stop — every kernel of later iterations returns at entry
    int stop_reason;   // 0 running, 1 max_iters, 2 tolerance, 3 diverged
    int diverged_iter; // first iteration whose audit failed, -1 if none
    int rows;          // trace rows written
    int audit;         // objective audit / trace active
    int check_diverge; // lipschitz step rule: monotone surrogate check
    int tol_kind;      // 0 none, 1 surrogate relative decrease, 2 relative step
    int fista;         // momentum on
    int refresh_inner; // per_inner weights (needs the previous iterate for after_{i-1})
    int done_y;        // stop flag of the y-forward pass: raised by the z pass that
                       // first sees `done`, so the last y-forward still runs
    double tol;
    double audit_slack; // relative slack of the monotone check (1e-9 in the reference)
    double step;        // l_r (constant within one m_step)
    double before[7];   // before_i of the iteration being audited (saved by finalize)
    double last_rel;    // last tolerance measure
    double step_max;    // largest ||x_{k+1} - x_k|| seen (tol_kind 2 normaliser)
    int restart;        // FISTA with gradient-based adaptive restart (momentum 2)
    int mom_base;       // iteration of the last restart: theta index = iter - mom_base
    int restarts;       // restarts taken
};

// a value the compiler cannot see through (forces recomputation of addresses
// derived from it instead of keeping them live in registers)
template <typename T> __device__ __forceinline__ T* opaque(T* p) {
    asm volatile("" : "+l"(p));
    return p;
}
__device__ __forceinline__ size_t opaque(size_t v) {
    asm volatile("" : "+l"(v));
    return v;
}
__device__ __forceinline__ int opaque(int v) {
    asm volatile("" : "+r"(v));
    return v;
}

#ifndef CM_PDL_EARLY
#define CM_PDL_EARLY 0  // trigger at CTA start (measured slower: dependents hold SM slots)
#endif
// programmatic dependent launch (PDL): the next kernel in the stream may be
// scheduled once every CTA of this one has triggered; it must wait for this
// grid's completion (and memory) before reading anything this grid wrote.
// Both are no-ops for a kernel launched without the PDL attribute.
__device__ __forceinline__ void pdl_trigger() {
#if CM_PDL_EARLY
    asm volatile("griddepcontrol.launch_dependents;");
#endif
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ int ld_done(const DevState* st) {
    return *((volatile const int*)&st->done);
}

// ---- reductions -------------------------------------------------------------
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum of NV doubles per thread; result valid in thread 0. scratch
// must hold 32*NV doubles.
// Sum over the first `width` lanes of a warp, valid in lane 0; safe when the
// warp is partial (blocks whose size is not a multiple of 32: radix-5/7 plans
// such as 10 threads per CTA at side 100). Lanes past `width` are never read.
__device__ __forceinline__ double warp_sum_partial(double v, int width) {
    const int lane = threadIdx.x & 31;
    const unsigned mask = width >= 32 ? 0xffffffffu : ((1u << width) - 1u);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_down_sync(mask, v, o);
        if (lane + o < width) v += t;
    }
    return v;
}

template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    if (blockDim.x & 31) {  // a partial last warp: guarded tree, fixed order
        const int width = min(32, (int)blockDim.x - 32 * wid);
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = warp_sum_partial(v[q], width);
        __syncthreads();
        if (lane == 0)
#pragma unroll
            for (int q = 0; q < NV; ++q) scratch[wid * NV + q] = v[q];
        __syncthreads();
        if (wid == 0) {
#pragma unroll
            for (int q = 0; q < NV; ++q) {
                double s = lane < nw ? scratch[lane * NV + q] : 0.0;
                v[q] = warp_sum_partial(s, min(32, (int)blockDim.x));
            }
        }
        return;
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) scratch[wid * NV + q] = v[q];
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int q = 0; q < NV; ++q) {
            double s = lane < nw ? scratch[lane * NV + q] : 0.0;
            v[q] = warp_sum(s);
        }
    }
}

} // namespace cm
