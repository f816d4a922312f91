// x-line real transforms (sm_100a): C2R of the packed half spectrum into the
// data gradient g = Re ifft3(...) / L, and R2C of a real volume into the packed
// half spectrum. One group of TX threads per line (warp-synchronous), lines
// loaded straight into registers (t + TX*m order: coalesced), registers out.
//
// A real line of N samples is transformed as N/2 complex samples
// z(p) = x(2p) + i x(2p+1); the split / merge with the mate h <-> N/2 - h uses
// one shared-memory exchange. The x-Nyquist value X(N/2) is packed into the
// imaginary part of column 0 (kernels.cuh layout).
#pragma once

#include <type_traits>

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"

namespace cm {

#ifndef CM_XFFT_E16
#define CM_XFFT_E16 1
#endif
#ifndef CM_XFFT_MINB
#define CM_XFFT_MINB 0
#endif

// x lines favour fewer, wider stages (radix-16): one exchange for 256 points
__host__ __device__ constexpr int xelems_for(int LEN) {
    return (CM_XFFT_E16 && LEN >= 256 && (LEN & (LEN - 1)) == 0) ? 16 : elems_for(LEN);
}

template <typename R, int N> struct XGeo {
    static constexpr int Nh = N / 2;
    static constexpr int E = xelems_for(Nh);
    static constexpr int T = Nh / E;
    static constexpr int LPC = (256 / T) < 1 ? 1 : (256 / T);  // lines per CTA
    static constexpr int NT = LPC * T < 32 ? 32 : LPC * T;
    static constexpr int LPCB = NT / T;
    static constexpr int PADX = (Nh + (Nh >> 3) + 2) / 2 * 2;
    static constexpr size_t SMEM = sizeof(Cx<R>) * (N + (size_t)LPCB * PADX) + packed_tw_bytes<R>(N, 1);
    static constexpr int NB = (N * N + LPC - 1) / LPC;
    // resident CTAs per SM the register budget must allow (>= 24 warps per SM)
    static constexpr int MINB = (CM_XFFT_MINB > 0) ? CM_XFFT_MINB : (NT <= 256 && sizeof(R) == 4 ? 3 : 1);
};

template <typename R> struct XfParams {
    using C = Cx<R>;
    C* S;
    R* real;            // C2R: g out (scaled by `scale`); R2C: volume in
    const C* twN;
    const float4* tw4;  // packed table of the transform direction (fp32)
    const int* stop;    // &st->done (C2R) / &st->done_y (R2C) or null
    double scale;
    int nlines;         // lines to transform (N*N, or NK*N on a z-slab rank)
};

#ifndef CM_XFFT_TWPOW
#define CM_XFFT_TWPOW 1
#endif

// x-line twiddles: powers of one table entry per stage in fp32 (bank conflicts,
// cm_common.cuh TwPow), the plain table in fp64
template <typename R, bool FWD>
__device__ __forceinline__ auto xline_tw(const Cx<R>* plain, const float4* packed) {
    if constexpr (sizeof(R) == 4 && CM_XFFT_TWPOW) {
        (void)packed;
        return TwPow<Cx<R>, FWD>{plain};
    } else {
        return tw_src<R, FWD>(plain, packed);
    }
}

// DIR 0: C2R (S -> real * scale), DIR 1: R2C (real -> S)
template <typename R, int N, int DIR>
__global__ void __launch_bounds__(XGeo<R, N>::NT, XGeo<R, N>::MINB) xfft_kernel(XfParams<R> p) {
    using X = XGeo<R, N>;
    using C = Cx<R>;
    constexpr int Nh = X::Nh, E = X::E, T = X::T;
    pdl_trigger();
    pdl_wait();
    if (p.stop && *((volatile const int*)p.stop)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* lines = tw + N;
    float4* tw4 = reinterpret_cast<float4*>(lines + X::LPCB * X::PADX);
    stage_table(tw, p.twN, N);
    if constexpr (use_packed_tw<R>()) stage_table(tw4, p.tw4, N);
    __syncthreads();
    const int lg = threadIdx.x / T, t = threadIdx.x % T;
    C* buf = lines + lg * X::PADX;
    const PadAddr pad{};
    // a line's T threads inside one warp: warp barriers; T not dividing 32 (sides
    // with an odd factor in N/2 / E, e.g. 100 = 4 * 25) lets groups straddle
    // warps: block barriers (every thread runs the same sequence)
    using LineSync = std::conditional_t<(32 % T == 0), WarpSync, BlockSync>;
    const LineSync wsync{};
    // persistent: the twiddle table is staged once per CTA
    const int ngrp = (p.nlines + X::LPC - 1) / X::LPC;
    for (int grp = blockIdx.x; grp < ngrp; grp += gridDim.x) {
    const int line = grp * X::LPC + lg;
    const bool valid = (lg < X::LPC) && (line < p.nlines);
    C* Srow = p.S + (size_t)(valid ? line : 0) * Nh;
    R* xrow = p.real + (size_t)(valid ? line : 0) * N;
    C v[E];
    if constexpr (DIR == 0) {
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = valid ? Srow[t + T * m] : cx<C>(R(0), R(0));
        wsync();
#pragma unroll
        for (int m = 0; m < E; ++m) buf[pad(t + T * m)] = v[m];
        wsync();
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int hh = t + T * m;
            const C q = v[m];
            if (hh == 0) {
                v[m] = cx<C>(q.x + q.y, q.x - q.y);
            } else {
                const C qm = buf[pad(Nh - hh)];
                const C a = cx<C>(q.x + qm.x, q.y - qm.y);   // Q + conj(Qm)
                const C d = cx<C>(q.x - qm.x, q.y + qm.y);   // Q - conj(Qm)
                const C bb = cmulc(d, tw[hh]);               // * exp(+2 pi i h / N)
                v[m] = cx<C>(a.x - bb.y, a.y + bb.x);        // A + i B
            }
        }
        wsync();
        fft_regs<Nh, E, N, false>(v, t, buf, pad, xline_tw<R, false>(tw, tw4), wsync);
        const R sc = R(p.scale);
        if (valid)
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int pp = t + T * m;
                *reinterpret_cast<C*>(xrow + 2 * pp) = cx<C>(v[m].x * sc, v[m].y * sc);
            }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int pp = t + T * m;
            v[m] = valid ? *reinterpret_cast<const C*>(xrow + 2 * pp) : cx<C>(R(0), R(0));
        }
        wsync();
        fft_regs<Nh, E, N, true>(v, t, buf, pad, xline_tw<R, true>(tw, tw4), wsync);
        wsync();
#pragma unroll
        for (int m = 0; m < E; ++m) buf[pad(t + T * m)] = v[m];
        wsync();
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int hh = t + T * m;
            const C z = v[m];
            C out;
            if (hh == 0) {
                out = cx<C>(z.x + z.y, z.x - z.y);  // X(0) + i X(N/2)
            } else {
                const C zm = buf[pad(Nh - hh)];
                const C e = cx<C>(R(0.5) * (z.x + zm.x), R(0.5) * (z.y - zm.y));
                const C o = cx<C>(R(0.5) * (z.y + zm.y), R(-0.5) * (z.x - zm.x));
                out = cadd(e, cmul(o, tw[hh]));
            }
            if (valid) Srow[hh] = out;
        }
    }
    wsync();
    }
}

} // namespace cm
