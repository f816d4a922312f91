// Register-resident mixed-radix Stockham FFT engine (cuFFT-free).
//
// A sequence of length LEN is owned by T = LEN/E cooperating threads; thread
// t holds positions t + T*m (m < E) in registers. Every Stockham stage
// (radix R | E, Ns = product of earlier radices) reads exactly the thread's
// own positions, so the only data movement is one shared-memory exchange
// between consecutive stages; the first stage reads and the last stage writes
// the natural order directly, which keeps global loads and stores coalesced
// (consecutive threads -> consecutive positions or columns).
//
// Twiddles come from a shared-memory table tw[x] = exp(-2 pi i x / TWN)
// (TWN = table length, a multiple of LEN); the inverse uses conj.
// Radices: 16, 8, 4, 2 (compile-time split-in-half DIT with constant
// twiddles), 3, 5 and 7 (symmetric-pair odd DFTs).
#pragma once

#include <type_traits>

#include "cm_common.cuh"

namespace cm {

__host__ __device__ constexpr int pick_radix(int rem, int E) {
    return (rem % 16 == 0 && E % 16 == 0)   ? 16
           : (rem % 8 == 0 && E % 8 == 0)   ? 8
           : (rem % 4 == 0 && E % 4 == 0)   ? 4
           : (rem % 2 == 0 && E % 2 == 0)   ? 2
           : (rem % 3 == 0 && E % 3 == 0)   ? 3
           : (rem % 5 == 0 && E % 5 == 0)   ? 5
           : (rem % 7 == 0 && E % 7 == 0)   ? 7
                                            : 0;
}

__host__ __device__ constexpr int radix_at(int LEN, int E, int s) {
    int rem = LEN;
    for (int i = 0; i < s; ++i) rem /= pick_radix(rem, E);
    return pick_radix(rem, E);
}

__host__ __device__ constexpr int n_stages(int LEN, int E) {
    int rem = LEN, s = 0;
    while (rem > 1) {
        const int r = pick_radix(rem, E);
        if (r == 0) return -1;
        rem /= r;
        ++s;
    }
    return s;
}

// exp(-2 pi i k / 16) components, k = 0..15
__host__ __device__ constexpr double kCos16(int k) {
    constexpr double c[16] = {1.0,
                              0.92387953251128675613,
                              0.70710678118654752440,
                              0.38268343236508977173,
                              0.0,
                              -0.38268343236508977173,
                              -0.70710678118654752440,
                              -0.92387953251128675613,
                              -1.0,
                              -0.92387953251128675613,
                              -0.70710678118654752440,
                              -0.38268343236508977173,
                              0.0,
                              0.38268343236508977173,
                              0.70710678118654752440,
                              0.92387953251128675613};
    return c[k & 15];
}
__host__ __device__ constexpr double kSin16(int k) { return kCos16(k + 12); } // sin(x) = cos(x - pi/2)

// z * exp(-+2 pi i Q/R) for compile-time Q, R (R | 16)
template <int R, int Q, bool FWD, typename C>
__device__ __forceinline__ C tw_const(C z) {
    constexpr int k = (Q * (16 / R)) & 15;
    using Rt = decltype(C::x);
    if constexpr (k == 0) {
        return z;
    } else if constexpr (k == 4) {
        return cmul_mi<FWD>(z);  // exp(-i pi/2) = -i
    } else if constexpr (k == 8) {
        return cx<C>(-z.x, -z.y);
    } else if constexpr (k == 12) {
        return cmul_mi<!FWD>(z);
    } else {
        constexpr double c = kCos16(k);
        constexpr double s = FWD ? -kSin16(k) : kSin16(k); // exp(-i a): (cos a, -sin a)
        if constexpr (sizeof(Rt) == 4) {
            return __ffma2_rn(make_float2(z.y, z.y), make_float2(float(-s), float(c)),
                              __fmul2_rn(make_float2(z.x, z.x), make_float2(float(c), float(s))));
        } else {
            return cx<C>(z.x * Rt(c) - z.y * Rt(s), z.x * Rt(s) + z.y * Rt(c));
        }
    }
}

template <int R, bool FWD, typename C> struct Dft;

template <bool FWD, typename C> struct Dft<1, FWD, C> {
    static __device__ __forceinline__ void run(C (&)[1]) {}
};

template <bool FWD, typename C> struct Dft<2, FWD, C> {
    static __device__ __forceinline__ void run(C (&u)[2]) {
        const C a = u[0], b = u[1];
        u[0] = cadd(a, b);
        u[1] = csub(a, b);
    }
};

template <bool FWD, typename C> struct Dft<3, FWD, C> {
    static __device__ __forceinline__ void run(C (&u)[3]) {
        using Rt = decltype(C::x);
        const Rt s3 = Rt(FWD ? -0.86602540378443864676 : 0.86602540378443864676);
        const C a = u[0];
        const C sp = cadd(u[1], u[2]);
        const C dm = csub(u[1], u[2]);
        const C m = cx<C>(a.x - Rt(0.5) * sp.x, a.y - Rt(0.5) * sp.y);
        // i * s3 * dm = (-s3 dm.y, s3 dm.x)
        const C r = cx<C>(-s3 * dm.y, s3 * dm.x);
        u[0] = cadd(a, sp);
        u[1] = cadd(m, r);
        u[2] = csub(m, r);
    }
};

// odd prime radix P in {5, 7}: y_k = x0 + sum_j cos(2 pi jk/P) (x_j + x_{P-j})
//                                  -+ i sum_j sin(2 pi jk/P) (x_j - x_{P-j})
// (pairs j, P-j share the cosine and flip the sine; (P-1)^2/2 real FMAs per
// component instead of (P-1)^2)
__host__ __device__ constexpr double odd_cos(int P, int m) {
    return P == 5 ? (m == 1 ? 0.30901699437494742410 : -0.80901699437494742410)
                  : (m == 1 ? 0.62348980185873353053 : m == 2 ? -0.22252093395631440429
                                                              : -0.90096886790241912624);
}
__host__ __device__ constexpr double odd_sin(int P, int m) {
    return P == 5 ? (m == 1 ? 0.95105651629515357212 : 0.58778525229247312917)
                  : (m == 1 ? 0.78183148246802980871 : m == 2 ? 0.97492791218182360702
                                                              : 0.43388373911755812048);
}
template <int P, bool FWD, typename C> struct DftOdd {
    static __device__ __forceinline__ void run(C (&u)[P]) {
        using Rt = decltype(C::x);
        constexpr int H = (P - 1) / 2;
        C a[H + 1], b[H + 1];
#pragma unroll
        for (int j = 1; j <= H; ++j) {
            a[j] = cadd(u[j], u[P - j]);
            b[j] = csub(u[j], u[P - j]);
        }
        C y0 = u[0];
#pragma unroll
        for (int j = 1; j <= H; ++j) y0 = cadd(y0, a[j]);
        C out[P];
        out[0] = y0;
#pragma unroll
        for (int k = 1; k <= H; ++k) {
            Rt tx = u[0].x, ty = u[0].y, vx = Rt(0), vy = Rt(0);
#pragma unroll
            for (int j = 1; j <= H; ++j) {
                const int m = (j * k) % P;  // cos / sin of 2 pi m / P, m folded into 1..H
                const bool flip = m > H;
                const int mm = flip ? P - m : m;
                const Rt cc = Rt(odd_cos(P, mm));
                const Rt ss = flip ? Rt(-odd_sin(P, mm)) : Rt(odd_sin(P, mm));
                tx += cc * a[j].x;
                ty += cc * a[j].y;
                vx += ss * b[j].x;
                vy += ss * b[j].y;
            }
            // forward: y_k = t - i v, y_{P-k} = t + i v (inverse: signs swapped)
            const C iv = cx<C>(-vy, vx);  // i v
            out[k] = FWD ? cx<C>(tx - iv.x, ty - iv.y) : cx<C>(tx + iv.x, ty + iv.y);
            out[P - k] = FWD ? cx<C>(tx + iv.x, ty + iv.y) : cx<C>(tx - iv.x, ty - iv.y);
        }
#pragma unroll
        for (int k = 0; k < P; ++k) u[k] = out[k];
    }
};
template <bool FWD, typename C> struct Dft<5, FWD, C> {
    static __device__ __forceinline__ void run(C (&u)[5]) { DftOdd<5, FWD, C>::run(u); }
};
template <bool FWD, typename C> struct Dft<7, FWD, C> {
    static __device__ __forceinline__ void run(C (&u)[7]) { DftOdd<7, FWD, C>::run(u); }
};

// power-of-two radix: decimation in time split into even / odd halves
template <int R, bool FWD, typename C> struct Dft {
    static_assert(R == 4 || R == 8 || R == 16, "unsupported radix");
    template <int Q>
    static __device__ __forceinline__ void combine(C (&u)[R], const C (&e)[R / 2],
                                                   const C (&o)[R / 2]) {
        if constexpr (Q < R / 2) {
            const C t = tw_const<R, Q, FWD>(o[Q]);
            u[Q] = cadd(e[Q], t);
            u[Q + R / 2] = csub(e[Q], t);
            combine<Q + 1>(u, e, o);
        }
    }
    static __device__ __forceinline__ void run(C (&u)[R]) {
        C e[R / 2], o[R / 2];
#pragma unroll
        for (int r = 0; r < R / 2; ++r) {
            e[r] = u[2 * r];
            o[r] = u[2 * r + 1];
        }
        Dft<R / 2, FWD, C>::run(e);
        Dft<R / 2, FWD, C>::run(o);
        combine<0>(u, e, o);
    }
};

// ---- the engine -------------------------------------------------------------
// Addr: functor mapping a sequence position p to a shared-memory element
// offset (e.g. padded line layout, or [p][column] tile layout).
// Sync: functor performing the barrier that covers all threads of a sequence.
template <int LEN, int E, int TWN, bool FWD, int SI, int NS>
struct FftStage {
    template <typename C, typename Addr, typename Tw, typename Sync>
    static __device__ __forceinline__ void run(C (&v)[E], int t, C* buf, const Addr& addr,
                                               const Tw& tw, const Sync& sync) {
        constexpr int R = radix_at(LEN, E, SI);
        static_assert(R > 0, "LEN/E have no radix plan");
        constexpr int Q = E / R;
        constexpr int T = LEN / E;
        constexpr bool LAST = (NS * R == LEN);
        constexpr int TWSTEP = (LEN / (NS * R)) * (TWN / LEN);
#pragma unroll
        for (int q = 0; q < Q; ++q) {
            const int j = t + T * q;
            const int k = (NS == 1) ? 0 : (j % NS);
            C u[R];
#pragma unroll
            for (int r = 0; r < R; ++r) u[r] = v[q + r * Q];
            if constexpr (NS > 1) {
                if constexpr (tw_has_pow<Tw>::value && R >= 4) {
                    C wp[R];
                    wp[1] = tw.get(k * TWSTEP);
#pragma unroll
                    for (int r = 2; r < R; ++r)
                        wp[r] = (r % 2 == 0) ? cmul(wp[r / 2], wp[r / 2]) : cmul(wp[r - 1], wp[1]);
#pragma unroll
                    for (int r = 1; r < R; ++r) u[r] = cmul(u[r], wp[r]);
                } else {
#pragma unroll
                    for (int r = 1; r < R; ++r) u[r] = tw.mul(u[r], r * k * TWSTEP);
                }
            }
            Dft<R, FWD, C>::run(u);
            if constexpr (LAST) {
#pragma unroll
                for (int r = 0; r < R; ++r) v[q + r * Q] = u[r];
            } else {
                const int base = (NS == 1) ? j * R : (j / NS) * NS * R + k;
#pragma unroll
                for (int r = 0; r < R; ++r) buf[addr(base + r * NS)] = u[r];
            }
        }
        if constexpr (!LAST) {
            sync();
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = buf[addr(t + T * m)];
            sync();
            FftStage<LEN, E, TWN, FWD, SI + 1, NS * R>::run(v, t, buf, addr, tw, sync);
        }
    }
};

// tw: a twiddle source (TwPlain / TwPacked) of direction FWD, or a plain table
template <int LEN, int E, int TWN, bool FWD, typename C, typename Addr, typename Tw,
          typename Sync>
__device__ __forceinline__ void fft_regs(C (&v)[E], int t, C* buf, const Addr& addr,
                                         const Tw& tw, const Sync& sync) {
    static_assert(LEN % E == 0, "E must divide LEN");
    static_assert(TWN % LEN == 0, "twiddle table length must be a multiple of LEN");
    if constexpr (std::is_pointer<Tw>::value) {
        const TwPlain<C, FWD> src{tw};
        if constexpr (LEN > 1) FftStage<LEN, E, TWN, FWD, 0, 1>::run(v, t, buf, addr, src, sync);
    } else {
        if constexpr (LEN > 1) FftStage<LEN, E, TWN, FWD, 0, 1>::run(v, t, buf, addr, tw, sync);
    }
}

// Elements per thread for lengths with a factor 5 or 7: every distinct odd
// prime of LEN once (a radix-R stage needs R | E) times the largest power of
// two dividing LEN that keeps E <= 32
__host__ __device__ constexpr int elems_57(int LEN) {
    const int f = (LEN % 3 == 0 ? 3 : 1) * (LEN % 5 == 0 ? 5 : 1) * (LEN % 7 == 0 ? 7 : 1);
    int p2 = 1;
    while (LEN % (2 * p2) == 0 && f * 2 * p2 <= 32) p2 *= 2;
    return f * p2;
}
// Elements per thread for a transform of length LEN.
__host__ __device__ constexpr int elems_for(int LEN) {
    return LEN <= 24 ? LEN
           : (LEN % 5 == 0 || LEN % 7 == 0) ? elems_57(LEN)
           : (LEN % 3 == 0) ? (LEN >= 192 ? 24 : 12)
           : (LEN >= 512 ? 16 : 8);
}

#ifndef CM_PAD_SHIFT
#define CM_PAD_SHIFT 4
#endif
struct PadAddr {  // line layout, one pad element every CM_PAD_SHIFT^2 (bank spread)
    // 16: the radix-16 exchange writes positions 16 t + r of 16 lanes -> 17 t + r,
    // distinct banks for 8-byte elements (every 8 left a 2-way conflict)
    __device__ __forceinline__ int operator()(int p) const { return p + (p >> CM_PAD_SHIFT); }
};
struct ColAddr {  // [position][column] tile layout
    int tw, col;
    __device__ __forceinline__ int operator()(int p) const { return p * tw + col; }
};
struct WarpSync {
    __device__ __forceinline__ void operator()() const { __syncwarp(); }
};
struct BlockSync {
    __device__ __forceinline__ void operator()() const { __syncthreads(); }
};

} // namespace cm
