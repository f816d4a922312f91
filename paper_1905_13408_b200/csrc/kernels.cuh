// M-step solver kernels for sm_100a. See DESIGN.md for the schedule.
//
// Storage (real-space, x fastest, flat (k*N + j)*N + i as volume.hpp:13):
//   x      R[N][N][N]
// Half spectrum, PACKED (Nh = N/2 columns per row):
//   S      C[N][N][Nh]   column 0 holds X(0) + i X(Nh) of the x-transform,
//                        i.e. after the y/z transforms F(0,b,c) + i F(Nh,b,c)
//   W      R[N][N][Nh] + Wn R[N][N]   (h = Nh plane stored separately)
//   Yh     C[N][N][Nh] + Yn C[N][N]   Yh = (-1)^(a+b+c) * Hermitian part of Y
//
// Per iteration i (SURVEY §8(d) canonical 4-kernel schedule):
//   K3  z-forward, fit partials, G = W.F - Yh, z-inverse        (zpass_kernel)
//   K4  y-inverse                                               (ypass_kernel<false>)
//   K1  x C2R -> g; weights + Huber-TV stencil + ISTA/FISTA update + prox
//       + objective partials; x R2C of x_{i+1}                   (xline_kernel)
//   FIN fixed-order reduction of partials, trace row, audit     (finalize_kernel)
//   K2  y-forward                                               (ypass_kernel<true>)
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"

namespace cm {

// line-kernel modes of the component entry points and the audit epilogue (the
// solver's per-iteration sweep is stencil2/stencil; transforms are xfft/ypass/zpass)
enum XMode { XM_OBJ = 2, XM_TVGRAD = 4, XM_WEIGHTS = 5 };
enum ZMode { ZM_FULL = 0, ZM_FIT = 1, ZM_FWD = 2 };

constexpr int NP1 = 12; // xline partial slots (11: FISTA restart test)
constexpr int NP3 = 2;  // zpass partial slots

// ---- compile-time geometry ----------------------------------------------------
__host__ __device__ constexpr int pow2_divisor_le(int v, int cap) {
    int t = 1;
    while (t * 2 <= cap && v % (t * 2) == 0) t *= 2;
    return t;
}

#ifndef CM_Y_SMEM_CAP_KB
#define CM_Y_SMEM_CAP_KB 96
#endif
#ifndef CM_Y_TWMAX
#define CM_Y_TWMAX 16  // columns per y tile (128-byte rows in fp32)
#endif
// plans with >= 24 elements per thread (radix-3/5/7 sides): at most
// CM_Y_NT_E24 threads per y / z tile, two CTAs per SM (128 registers). The
// 512-thread tiles of 768^3 were held to 64 registers and spilled: z pass 2.79
// -> 1.86 ms, y passes 1.17 -> 0.90-0.95 ms (profiles/r2_ab_e24.txt)
#ifndef CM_Y_NT_E24
#define CM_Y_NT_E24 256
#endif
#ifndef CM_Y_MINB_E24
#define CM_Y_MINB_E24 2
#endif
#ifndef CM_Z_MINB_E24
#define CM_Z_MINB_E24 2
#endif

template <typename R, int N> struct Geo {
    using C = Cx<R>;
    static constexpr int Nh = N / 2;
    // x lines: transform length Nh
    static constexpr int EX = elems_for(Nh);
    static constexpr int TX = Nh / EX;
    static constexpr int LPC = (256 / TX) < 1 ? 1 : (256 / TX);   // lines per CTA
    static constexpr int PADX = Nh + (Nh >> 3) + 1;                 // padded line buffer (complex)
    // y / z columns: transform length N
    static constexpr int EY = elems_for(N);
    static constexpr int TY = N / EY;
    static constexpr int SMEM_CAP = CM_Y_SMEM_CAP_KB * 1024; // per tile buffer budget (bytes)
    static constexpr int TWY_CAP = (SMEM_CAP / (N * (int)sizeof(C))) < 1 ? 1 : (SMEM_CAP / (N * (int)sizeof(C)));
    static constexpr int TWMAX_ = (EY >= 24 && CM_Y_NT_E24 / TY < CM_Y_TWMAX)
                                      ? (CM_Y_NT_E24 / TY < 1 ? 1 : CM_Y_NT_E24 / TY)
                                      : CM_Y_TWMAX;
    static constexpr int TWY_LIM = (TWMAX_ < (1024 / TY) ? TWMAX_ : (1024 / TY));
    static constexpr int TWY = pow2_divisor_le(Nh, TWY_LIM < TWY_CAP ? TWY_LIM : TWY_CAP);
    static constexpr int TW3_LIM = (512 / TY) < 1 ? 1 : (512 / TY);
    static constexpr int TW3_CAP = TWY_CAP / 2 < 1 ? 1 : TWY_CAP / 2;
    static constexpr int TW3 = pow2_divisor_le(Nh, (16 < TW3_LIM ? 16 : TW3_LIM) < TW3_CAP ? (16 < TW3_LIM ? 16 : TW3_LIM) : TW3_CAP);
};

// ---- parameters -----------------------------------------------------------------
template <typename R> struct XParams {
    using C = Cx<R>;
    C* S;               // packed spectrum (in: G rows for SWEEP/DGRAD, out: rows of x_{i+1})
    const R* xcur;      // point of the stencil / gradient (x_i, or y_k for FISTA)
    const R* xprev;     // previous iterate for after_{i-1} weights (per_inner audit), or null
    const R* wsrc;      // weight source (per_inner: xcur; per_m_step: x_init)
    const R* anchor;    // restraint anchor
    const R* xold;      // FISTA: x_k (momentum base); null otherwise
    const R* wtvf;      // explicit w_tv field (component API), or null
    R* xnext;           // x_{i+1} out (SWEEP) / g or tv-gradient out (DGRAD/TVGRAD)
    R* ynext;           // FISTA: y_{k+1} out
    const C* twN;       // exp(-2 pi i q / N), q < N (global; staged into smem)
    const double* theta; // FISTA momentum per iteration (indexed by st->iter)
    double* part;       // [gridDim.x][NP1]
    DevState* st;
    double lr, alpha, beta, gamma, eps, eps_prime, mu, invL;
    int convex, audit, fista;
};

template <typename R> struct ZParams {
    using C = Cx<R>;
    C* S;
    const R* W;
    const R* Wn;
    const C* Yh;
    const C* Yn;
    const C* twN;
    double* part; // [grid][NP3]
    DevState* st;
};

// Spectrum layout of a y pass side: element (k, b, h) at
//   k*kstride + (b / nb)*sstride + (b % nb)*Nh + h
// natural [k][b][h]: kstride = N*Nh, nb = N, sstride = 0; destination-major
// [s][k][b_local][h] of a z-slab rank (the all-to-all send/receive layout):
// kstride = nb*Nh, sstride = NK*nb*Nh.
// z-slab ranks may also split the columns h into two halves stored one after
// the other (hh columns per row, the second half at +hstride) so that each half
// is transposed by its own all-to-all (comm/compute overlap, dist.cuh).
struct SpecLayout {
    long long kstride, sstride;
    int nb;
    float inv_nb;  // 1/nb: b = s nb + b_local without an integer division
    int hh;        // columns per stored row (Nh, or Nh/2 with split halves)
    long long hstride;
    __device__ __forceinline__ long long at(int k, int b, int h, int) const {
        // exact: (b + 1/2)/nb is at least 1/(2 nb) away from an integer, b < 2^12
        const int s = __float2int_rz(((float)b + 0.5f) * inv_nb);
        const int hq = h >= hh ? 1 : 0;
        return (long long)hq * hstride + (long long)k * kstride + (long long)s * sstride +
               (long long)(b - s * nb) * hh + (h - hq * hh);
    }
};
inline SpecLayout spec_layout(long long kstride, long long sstride, int nb, int hh,
                              long long hstride = 0) {
    return {kstride, sstride, nb, 1.0f / (float)nb, hh, hstride};
}

template <typename R> struct YParams {
    using C = Cx<R>;
    C* S;               // input spectrum
    const C* twN;
    const float4* tw4;  // packed table of the pass direction (fp32)
    const int* stop;    // &st->done (inverse pass) or &st->done_y (forward pass), or null
    C* Sout;            // output spectrum (may equal S), or null for in place
    SpecLayout lin, lout;
    int nplanes;        // planes k (N, or NK on a z-slab rank)
    int htile0, htiles; // column tiles [htile0, htile0 + htiles) (0, Nh/TWY: all)
};

template <typename C>
__device__ __forceinline__ void stage_table(C* dst, const C* src, int n) {
    for (int q = threadIdx.x; q < n; q += blockDim.x) dst[q] = src[q];
}

// twiddle source of a kernel: packed {w, i w} tables in fp32, plain table in fp64
template <typename R, bool FWD>
__device__ __forceinline__ auto tw_src(const Cx<R>* plain, const float4* packed) {
    if constexpr (sizeof(R) == 4 && CM_PACKED_TW) {
        return TwPacked{packed};
    } else {
        return TwPlain<Cx<R>, FWD>{plain};
    }
}
template <typename R> __host__ __device__ constexpr size_t packed_tw_bytes(int n, int tables) {
    return (sizeof(R) == 4 && CM_PACKED_TW) ? (size_t)16 * n * tables : 0;
}
template <typename R> __host__ __device__ constexpr bool use_packed_tw() { return sizeof(R) == 4 && CM_PACKED_TW; }

// ==================================================================================
// y pass: FFT along j for every (k, h) column. grid = (Nh/TWY, N)
// ==================================================================================
#ifndef CM_Y_PIPE
#define CM_Y_PIPE 1  // load the next tile while transforming this one (one CTA per SM)
#endif

// power-of-two sides >= 256 (16 elements per thread); radix-3 plans hold 24
template <int N> __host__ __device__ constexpr bool y_pipe() {
    return CM_Y_PIPE && N >= 256 && (N & (N - 1)) == 0 &&
           Geo<float, N>::TWY * Geo<float, N>::TY <= 512;  // two tiles in registers
}

template <typename R, int N, bool FWD, bool DM = false>
__global__ void __launch_bounds__(Geo<R, N>::TWY * Geo<R, N>::TY,
                                  (Geo<R, N>::TWY * Geo<R, N>::TY <= 512 && !y_pipe<N>())
                                      ? (Geo<R, N>::EY >= 24 ? CM_Y_MINB_E24 : 2)
                                      : 1)
ypass_kernel(YParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    pdl_trigger();
    pdl_wait();
    if (p.stop && *((volatile const int*)p.stop)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* buf = tw + N;
    float4* tw4 = reinterpret_cast<float4*>(buf + N * G::TWY);
    if constexpr (use_packed_tw<R>()) stage_table(tw4, p.tw4, N);
    else stage_table(tw, p.twN, N);
    const int col = threadIdx.x % G::TWY;
    const int t = threadIdx.x / G::TWY;
    // persistent over (column tile, plane): the twiddle table is staged once
    const int NTX = p.htiles;
    const int ntiles = NTX * p.nplanes;
    if constexpr (y_pipe<N>()) {
        // software pipeline: the loads of the next tile are in flight during
        // this tile's transform (registers for both: one CTA per SM)
        const int stride = gridDim.x * gridDim.y;
        int tile = blockIdx.y * gridDim.x + blockIdx.x;
        auto load = [&](int tl, C (&dst)[G::EY]) {
            const int hh = (p.htile0 + tl % NTX) * G::TWY + col, kk = tl / NTX;
            if constexpr (!DM) {
                const C* b0 = p.S + (size_t)kk * p.lin.kstride + hh;
#pragma unroll
                for (int m = 0; m < G::EY; ++m) dst[m] = b0[(size_t)(t + G::TY * m) * G::Nh];
            } else {
#pragma unroll
                for (int m = 0; m < G::EY; ++m) dst[m] = p.S[p.lin.at(kk, t + G::TY * m, hh, G::Nh)];
            }
        };
        C vn[G::EY];
        if (tile < ntiles) load(tile, vn);
        for (; tile < ntiles; tile += stride) {
            C v[G::EY];
#pragma unroll
            for (int m = 0; m < G::EY; ++m) v[m] = vn[m];
            if (tile + stride < ntiles) load(tile + stride, vn);
            __syncthreads();
            fft_regs<N, G::EY, N, FWD>(v, t, buf, ColAddr{G::TWY, col}, tw_src<R, FWD>(tw, tw4),
                                       BlockSync{});
            const int hh = (p.htile0 + tile % NTX) * G::TWY + col, kk = tile / NTX;
            if constexpr (!DM) {
                C* base = p.S + (size_t)kk * p.lin.kstride + hh;
#pragma unroll
                for (int m = 0; m < G::EY; ++m) base[(size_t)(t + G::TY * m) * G::Nh] = v[m];
            } else {
                C* out = p.Sout ? p.Sout : p.S;
#pragma unroll
                for (int m = 0; m < G::EY; ++m) out[p.lout.at(kk, t + G::TY * m, hh, G::Nh)] = v[m];
            }
        }
        return;
    }
    for (int tile = blockIdx.y * gridDim.x + blockIdx.x; tile < ntiles; tile += gridDim.x * gridDim.y) {
    const int h = (p.htile0 + tile % NTX) * G::TWY + col;
    const int k = tile / NTX;
    C v[G::EY];
    if constexpr (!DM) {  // natural layout, in place
        C* base = p.S + (size_t)k * p.lin.kstride + h;
#pragma unroll
        for (int m = 0; m < G::EY; ++m) v[m] = base[(size_t)(t + G::TY * m) * G::Nh];
        __syncthreads();
        fft_regs<N, G::EY, N, FWD>(v, t, buf, ColAddr{G::TWY, col}, tw_src<R, FWD>(tw, tw4),
                                   BlockSync{});
#pragma unroll
        for (int m = 0; m < G::EY; ++m) base[(size_t)(t + G::TY * m) * G::Nh] = v[m];
    } else {  // z-slab rank: natural <-> destination-major (fused all-to-all packing)
#pragma unroll
        for (int m = 0; m < G::EY; ++m) v[m] = p.S[p.lin.at(k, t + G::TY * m, h, G::Nh)];
        __syncthreads();
        fft_regs<N, G::EY, N, FWD>(v, t, buf, ColAddr{G::TWY, col}, tw_src<R, FWD>(tw, tw4),
                                   BlockSync{});
        // store offsets computed here, not held live across the transform
        C* out = opaque(p.Sout ? p.Sout : p.S);
        const int ko = opaque(k), to = opaque(t), ho = opaque(h);
#pragma unroll
        for (int m = 0; m < G::EY; ++m) out[p.lout.at(ko, to + G::TY * m, ho, G::Nh)] = v[m];
    }
    }
}

// ==================================================================================
// x lines: C2R -> data gradient; fused stencil sweep; R2C of the new iterate.
// ==================================================================================
template <typename R> struct Vox {
    const R* x;
    int N;
    __device__ __forceinline__ R at(int i, int j, int k) const {
        return __ldg(x + ((size_t)k * N + j) * N + i);
    }
};

// ||D x|| at (i,j,k) with the replicate rule (gradient.cpp:7-24), given x there
template <typename R>
__device__ __forceinline__ void grad3(const Vox<R>& v, int i, int j, int k, R xc, R& d1, R& d2,
                                      R& d3) {
    d1 = i > 0 ? xc - v.at(i - 1, j, k) : R(0);
    d2 = j > 0 ? xc - v.at(i, j - 1, k) : R(0);
    d3 = k > 0 ? xc - v.at(i, j, k - 1) : R(0);
}

template <typename R> __device__ __forceinline__ R rnorm3(R a, R b, R c) {
    return sqrt(a * a + b * b + c * c);
}
template <typename R> __device__ __forceinline__ R huber(R g, R mu) {
    return g < mu ? g * g / (R(2) * mu) : g - mu / R(2);
}

template <typename R, int N, int MODE>
__global__ void __launch_bounds__(Geo<R, N>::LPC * Geo<R, N>::TX)
xline_kernel(XParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    constexpr int T = G::TX, LPC = G::LPC;
    if (p.st && ld_done(p.st)) return;
    __shared__ double red[32 * NP1];

    const int lg = threadIdx.x / T;  // line within CTA
    const int t = threadIdx.x % T;
    const int line = blockIdx.x * LPC + lg;
    const bool valid = line < N * N;
    const int j = valid ? line % N : 0;
    const int k = valid ? line / N : 0;

    double acc[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) acc[q] = 0.0;

    {
        const Vox<R> X{p.xcur, N};
        const Vox<R> Wv{p.wsrc, N};
        const bool same_w = (p.wsrc == p.xcur);
        const R eps = R(p.eps), epsp = R(p.eps_prime), mu = R(p.mu);
        const bool want_tv = (MODE == XM_TVGRAD);
        const bool audit = (MODE == XM_OBJ);
        // w_tv at a voxel whose own gradient norm is qn (regularizer.cpp:44-59)
        auto wtv_at = [&](int ii, int jj, int kk, R qn) -> R {
            if (p.convex) return R(1);
            if (p.wtvf) return __ldg(p.wtvf + ((size_t)kk * N + jj) * N + ii);
            if (same_w) return R(1) / (qn + epsp);
            R e1, e2, e3;
            grad3(Wv, ii, jj, kk, Wv.at(ii, jj, kk), e1, e2, e3);
            return R(1) / (rnorm3(e1, e2, e3) + epsp);
        };
        if (valid) {
            for (int i = t; i < N; i += T) {
                const size_t gi = (size_t)line * N + i;
                const R xc = X.at(i, j, k);
                R d1, d2, d3;
                grad3(X, i, j, k, xc, d1, d2, d3);
                const R gn = rnorm3(d1, d2, d3);
                const R wl1 = p.convex ? R(1)
                                       : R(1) / (fabs(same_w ? xc : Wv.at(i, j, k)) + eps);
                const R wtv = wtv_at(i, j, k, gn);
                if constexpr (MODE == XM_WEIGHTS) {
                    p.xnext[gi] = wl1;
                    p.ynext[gi] = wtv;
                    continue;
                }
                R tvg = R(0);
                if (want_tv) {
                    // D*(s Dx) with s = w_tv / max(mu, ||Dx||) (regularizer.cpp:72-85,
                    // adjoint gradient.cpp:29-64)
                    const R s0 = wtv / (mu > gn ? mu : gn);
                    tvg = s0 * (d1 + d2 + d3);
#pragma unroll
                    for (int ax = 0; ax < 3; ++ax) {
                        if ((ax == 0 && i == N - 1) || (ax == 1 && j == N - 1) ||
                            (ax == 2 && k == N - 1))
                            continue;
                        const int ii = i + (ax == 0), jj = j + (ax == 1), kk = k + (ax == 2);
                        const R xq = X.at(ii, jj, kk);
                        R q1, q2, q3;
                        grad3(X, ii, jj, kk, xq, q1, q2, q3);
                        const R qn = rnorm3(q1, q2, q3);
                        const R sq = wtv_at(ii, jj, kk, qn) / (mu > qn ? mu : qn);
                        tvg -= sq * (ax == 0 ? q1 : (ax == 1 ? q2 : q3));
                    }
                }
                if constexpr (MODE == XM_TVGRAD) {
                    p.xnext[gi] = tvg;
                    continue;
                }
                const R av = p.anchor ? __ldg(p.anchor + gi) : R(0);
                if (audit) {
                    const double ax = fabs((double)xc);
                    const double hb = (double)huber(gn, mu);
                    acc[0] += (double)wl1 * ax;
                    acc[1] += (double)wtv * hb;
                    acc[2] += (double)wtv * (double)gn;
                    // log-norms: the fp32 product mode evaluates the logs in fp32 (MUFU,
                    // ~1 ulp; fp64 log on every voxel made this epilogue 13% of HBM peak),
                    // the fp64 parity mode in fp64
                    if constexpr (sizeof(R) == 4) {
                        acc[3] += (double)__logf(fabsf(xc) + eps);
                        acc[4] += (double)__logf(gn + epsp);
                    } else {
                        acc[3] += (double)log(fabs(xc) + eps);
                        acc[4] += (double)log(gn + epsp);
                    }
                    const double dd = (double)xc - (double)av;
                    acc[5] += dd * dd;
                    if (p.xprev) {
                        const Vox<R> P{p.xprev, N};
                        const R pc = P.at(i, j, k);
                        R e1, e2, e3;
                        grad3(P, i, j, k, pc, e1, e2, e3);
                        const R pl1 = R(1) / (fabs(pc) + eps);
                        const R ptv = R(1) / (rnorm3(e1, e2, e3) + epsp);
                        acc[6] += (double)pl1 * ax;
                        acc[7] += (double)ptv * hb;
                        acc[8] += (double)ptv * (double)gn;
                    }
                }
            }
        }
    }

    if constexpr (MODE == XM_OBJ) {
        if (p.part) {
            block_sum<NP1>(acc, red);
            if (threadIdx.x == 0)
#pragma unroll
                for (int q = 0; q < NP1; ++q) p.part[(size_t)blockIdx.x * NP1 + q] = acc[q];
        }
    }
}

template <typename R, int N> struct YSmem {
    static constexpr size_t bytes =
        sizeof(Cx<R>) * (N + (size_t)N * Geo<R, N>::TWY) + packed_tw_bytes<R>(N, 1);
};

} // namespace cm
