// K1 — fused x-line C2R + reweighted Huber-TV / l1 proximal step + R2C (sm_100a).
//
// Persistent grid; each CTA walks tiles of TK x TJ x-lines (TK planes x TJ rows,
// whole lines of N voxels). Per tile:
//   1. C2R: every line's packed half spectrum G(h) -> data gradient g (line buffer)
//   2. sweep, in i-chunks of CI voxels:
//        stage x (tile + 1-voxel halo on every side) and x_prev (backward halo)
//        in shared memory; compute the TV dual scale
//            s(q) = w_tv(q) / max(mu, |Dx(q)|)        (regularizer.cpp:72-85)
//        ONCE per voxel of the tile box + forward halo; then per voxel
//            tvg = s(p) (d1+d2+d3) - sum_a [p_a < N-1] s(p+e_a) (x(p+e_a) - x(p))
//        (= D*(s Dx), gradient.cpp:29-64), the ISTA/FISTA update, the
//        soft-threshold prox and the objective partials (before_i and, from
//        x_prev, the weight-dependent terms of after_{i-1})
//   3. R2C of the new iterate into the same spectrum rows.
// DRAM: spectrum rows r+w, x, anchor, x_next (+x_prev in audit per_inner,
// +w_tv field in per_m_step); the halo re-reads hit L2.
#pragma once

#include <type_traits>

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "tma.cuh"

#ifndef CM_SWEEP_TJ
#define CM_SWEEP_TJ 4
#endif

namespace cm {

__host__ __device__ constexpr int largest_divisor_le(int n, int cap) {
    int d = 1;
    for (int q = 1; q <= cap && q <= n; ++q)
        if (n % q == 0) d = q;
    return d;
}

template <typename R, int N> struct SwGeo {
    using C = Cx<R>;
    static constexpr int Nh = N / 2;
    static constexpr int EX = elems_for(Nh);
    static constexpr int TX = Nh / EX;          // threads per line in the FFT phases
    static constexpr int TJ = largest_divisor_le(N, CM_SWEEP_TJ);
    static constexpr int TK = 2;
    static constexpr int LPC = TJ * TK;         // lines per tile
    static constexpr int NT0 = LPC * TX;
    static constexpr int NT = NT0 < 64 ? 64 : NT0;  // threads per CTA
    static constexpr int NW = NT / 32;
    static constexpr int LPCB = NT / TX;        // line buffers (>= LPC; extra groups idle)
    static constexpr int CI = largest_divisor_le(N, 128);  // sweep chunk along x
    static constexpr int NCH = N / CI;
    static constexpr int PADX = (Nh + (Nh >> 3) + 2) / 2 * 2;  // even: 16-byte aligned lines
    // staged rows: element c (global i = i0 - 1 + c) at column c + 3, so the
    // body [i0, i0+CI) starts 16-byte aligned at column 4
    static constexpr int XSW = ((CI + 2 + 3) + 3) / 4 * 4;   // staged x row width
    static constexpr int XSR = (TK + 2) * (TJ + 2);         // staged x rows
    static constexpr int XPW = XSW;
    static constexpr int XPR = (TK + 1) * (TJ + 1);
    // fp32 with 128-voxel chunks: every lane owns 4 consecutive voxels (16-byte
    // shared / global accesses) and the x halo boxes arrive by TMA, double
    // buffered; other sizes and fp64 take the synchronous scalar path
    static constexpr bool V4 = (sizeof(R) == 4) && (CI == 128);
    static constexpr int SSW = V4 ? CI + 4 : CI + 1;
    static constexpr int SSR = (TK + 1) * (TJ + 1);
    static constexpr int NTILES = (N / TJ) * (N / TK);
    // TMA boxes
    static constexpr int GW = Nh < 256 ? Nh : 256;          // spectrum row box width
    static constexpr int NHB = Nh / GW;
    static constexpr uint32_t XBOX_BYTES = (uint32_t)(XSW * (TJ + 2) * (TK + 2) * sizeof(R));
    static constexpr uint32_t GBYTES = (uint32_t)(LPC * Nh * sizeof(C));
    // shared memory layout (bytes)
    static constexpr size_t al(size_t v, size_t a) { return (v + a - 1) / a * a; }
    static constexpr size_t OFF_LINES = al(sizeof(C) * N, 128);
    static constexpr size_t OFF_XS = al(OFF_LINES + sizeof(C) * (size_t)LPCB * PADX, 128);
    static constexpr size_t XS_BYTES = sizeof(R) * (size_t)XSR * XSW;
    static constexpr size_t OFF_XP = al(OFF_XS + (V4 ? 2 : 1) * XS_BYTES, 128);
    static constexpr size_t OFF_SS = al(OFF_XP + (V4 ? 0 : sizeof(R) * (size_t)XPR * XPW), 128);
    static constexpr size_t OFF_G = al(OFF_SS + sizeof(R) * (size_t)SSR * SSW, 128);
    static constexpr size_t OFF_RED = al(OFF_G + (V4 ? (size_t)GBYTES : 0), 128);
    static constexpr size_t OFF_BAR = al(OFF_RED + sizeof(double) * 32 * NP1, 16);
    static constexpr size_t SMEM = OFF_BAR + 4 * sizeof(uint64_t);
    static constexpr int MINB = (SMEM * 3 <= 220 * 1024 && NT <= 256) ? 3
                                : ((SMEM * 2 <= 220 * 1024 && NT <= 512) ? 2 : 1);
};

// fp32 product mode: single-MUFU approximations (rel. error ~1 ulp; the parity
// bar is 1e-5). fp64 parity mode: IEEE operations.
template <typename R> __device__ __forceinline__ R rcp_(R v);
template <> __device__ __forceinline__ float rcp_<float>(float v) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
template <> __device__ __forceinline__ double rcp_<double>(double v) { return 1.0 / v; }
template <typename R> __device__ __forceinline__ R sqrt_(R v);
template <> __device__ __forceinline__ float sqrt_<float>(float v) {
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v));
    return r;
}
template <> __device__ __forceinline__ double sqrt_<double>(double v) { return sqrt(v); }
template <typename R> __device__ __forceinline__ R log_(R v);
template <> __device__ __forceinline__ float log_<float>(float v) { return __logf(v); }
template <> __device__ __forceinline__ double log_<double>(double v) { return log(v); }

// Stage rows (k0 + kk, j0 + jj), kk in [-1, NRK-2], jj in [-1, RW-2] (RW rows
// per plane), global i in [i0 - 1, i0 + CI - (full ? 0 : 1)] into dst[row][c + 3]
// (c = i - i0 + 1): the body [i0, i0 + CI) as 16-byte vectors, halos scalar.
// Out-of-grid elements are 0 (never used: the replicate rule masks them).
template <typename R, int N, int CI, int RW>
__device__ __forceinline__ void stage_rows(R* dst, int nrows, const R* src, int k0, int j0,
                                           int i0, bool full, int wid, int lane) {
    constexpr int W = ((CI + 2 + 3) + 3) / 4 * 4;
    const int nw = blockDim.x >> 5;
    for (int r = wid; r < nrows; r += nw) {
        const int kk = r / RW - 1, jj = r - (r / RW) * RW - 1;
        const int gk = k0 + kk, gj = j0 + jj;
        const bool rok = gk >= 0 && gk < N && gj >= 0 && gj < N;
        const R* row = src + ((size_t)(rok ? gk : 0) * N + (rok ? gj : 0)) * N;
        R* d = dst + r * W;
        if constexpr ((CI % 4 == 0) && (N % 4 == 0)) {
            using V = typename std::conditional<sizeof(R) == 4, float4, double2>::type;
            constexpr int PER = 16 / sizeof(R);
            for (int v = lane; v < CI / PER; v += 32) {
                V val;
                if (rok) val = __ldg(reinterpret_cast<const V*>(row + i0) + v);
                else val = V{};
                *reinterpret_cast<V*>(d + 4 + v * PER) = val;
            }
        } else {
            for (int c = lane; c < CI; c += 32) d[4 + c] = rok ? __ldg(row + i0 + c) : R(0);
        }
        if (lane == 0) d[3] = (rok && i0 > 0) ? __ldg(row + i0 - 1) : R(0);
        if (lane == 1 && full) d[4 + CI] = (rok && i0 + CI < N) ? __ldg(row + i0 + CI) : R(0);
    }
}

template <typename R> struct SweepParams {
    using C = Cx<R>;
    C* S;
    const R* xcur;      // stencil / gradient point (x_i, FISTA: y_k)
    const R* xprev;     // x_{i-1} for the weights of after_{i-1} (per_inner audit), or null
    const R* wtvf;      // per_m_step: w_tv field of the weight source, or null
    const R* wl1src;    // per_m_step: weight source for w_l1 (null -> from xcur)
    const R* anchor;
    const R* xold;      // FISTA x_k
    R* xnext;
    R* ynext;           // FISTA y_{k+1}
    const C* twN;
    const double* theta;
    double* part;       // [gridDim.x][NP1]
    DevState* st;
    double lr, alpha, beta, gamma, eps, eps_prime, mu, invL;
    int convex, audit, fista;
    int dbg;  // timing experiments only: bit0 skip C2R, bit1 skip R2C, bit2 skip staging,
              // bit3 skip s box, bit4 skip voxel math (results are then wrong)
};


// ---- fp32 4-voxel paths (V4) ---------------------------------------------------------
__device__ __forceinline__ float4 ld4(const float* q) { return *reinterpret_cast<const float4*>(q); }
__device__ __forceinline__ void st4(float* q, float a, float b, float c, float d) {
    *reinterpret_cast<float4*>(q) = make_float4(a, b, c, d);
}

// TV dual scale s = w_tv / max(mu, |Dx|) on the (TK+1) x (TJ+1) x (CI+1) box
template <int N, int TJ>
__device__ __forceinline__ void sbox_v4(float* SS, const float* XS, const float* wtvf, int convex,
                                        int k0, int j0, int i0, float mu, float epsp, int wid,
                                        int lane) {
    constexpr int CI = 128, XSW = ((CI + 2 + 3) + 3) / 4 * 4, SSW = CI + 4;
    constexpr int SSR = 3 * (TJ + 1);
    const int nw = blockDim.x >> 5;
    for (int r = wid; r < SSR; r += nw) {
        const int kk = r / (TJ + 1), jj = r - kk * (TJ + 1);
        const int gj = j0 + jj, gk = k0 + kk;
        const bool rok = gj < N && gk < N;
        const float* xr = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + 4;
        float* srow = SS + r * SSW;
        const float* wrow = (wtvf && rok) ? wtvf + ((size_t)gk * N + gj) * N + i0 : nullptr;
        const int ii = 4 * lane;
        float sv[4] = {0.f, 0.f, 0.f, 0.f};
        if (rok) {
            const float4 c4 = ld4(xr + ii), y4 = ld4(xr + ii - XSW),
                         z4 = ld4(xr + ii - (TJ + 2) * XSW);
            const float xm = xr[ii - 1];
            const float xc[4] = {c4.x, c4.y, c4.z, c4.w}, xl[4] = {xm, c4.x, c4.y, c4.z};
            const float xy[4] = {y4.x, y4.y, y4.z, y4.w}, xz[4] = {z4.x, z4.y, z4.z, z4.w};
            float wt[4] = {1.f, 1.f, 1.f, 1.f};
            if (wrow) {
                const float4 w4 = __ldg(reinterpret_cast<const float4*>(wrow + ii));
                wt[0] = w4.x; wt[1] = w4.y; wt[2] = w4.z; wt[3] = w4.w;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float d1 = (i0 + ii + c) > 0 ? xc[c] - xl[c] : 0.f;
                const float d2 = gj > 0 ? xc[c] - xy[c] : 0.f;
                const float d3 = gk > 0 ? xc[c] - xz[c] : 0.f;
                const float gn = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                const float w = convex ? 1.f : (wrow ? wt[c] : rcp_(gn + epsp));
                sv[c] = w * rcp_(mu > gn ? mu : gn);
            }
        }
        st4(srow + ii, sv[0], sv[1], sv[2], sv[3]);
        if (lane == 0) {  // forward halo ii = CI
            const int gi = i0 + CI;
            float s1 = 0.f;
            if (rok && gi < N) {
                const float* q = xr + CI;
                const float xc = q[0];
                const float d1 = xc - q[-1];
                const float d2 = gj > 0 ? xc - q[-XSW] : 0.f;
                const float d3 = gk > 0 ? xc - q[-(TJ + 2) * XSW] : 0.f;
                const float gn = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                const float w = convex ? 1.f : (wtvf ? __ldg(wtvf + ((size_t)gk * N + gj) * N + gi)
                                                     : rcp_(gn + epsp));
                s1 = w * rcp_(mu > gn ? mu : gn);
            }
            srow[CI] = s1;
        }
    }
}

// one x-line of 128 voxels of the tile: update, prox, partials (4 voxels per lane)
template <int N, int TJ>
__device__ __forceinline__ void voxels_v4(const SweepParams<float>& p, float (&fa)[NP1],
                                          const float* XS, const float* XP, const float* SS,
                                          float* lbuf, int gk, int gj, int kk, int jj, int i0,
                                          int lane, bool has_alpha, bool has_beta, float theta) {
    constexpr int CI = 128, XSW = ((CI + 2 + 3) + 3) / 4 * 4, XPW = XSW, SSW = CI + 4;
    const int ii = 4 * lane;
    const int gi0 = i0 + ii;
    const size_t gidx = ((size_t)gk * N + gj) * N + gi0;
    const float eps = float(p.eps), epsp = float(p.eps_prime), mu = float(p.mu);
    const float lr = float(p.lr), alpha = float(p.alpha), beta = float(p.beta);
    const float gamma = float(p.gamma), invL = float(p.invL);
    const float4 a4 = __ldg(reinterpret_cast<const float4*>(p.anchor + gidx));
    // global loads first (before any store) so their latency overlaps the math:
    // backward stencil of x_{i-1} (L1/L2) for the weights of after_{i-1}
    float4 p4 = make_float4(0.f, 0.f, 0.f, 0.f), py4 = p4, pz4 = p4;
    float pm = 0.f;
    if (p.audit && p.xprev) {
        const float* pr = p.xprev + gidx;
        p4 = __ldg(reinterpret_cast<const float4*>(pr));
        py4 = gj > 0 ? __ldg(reinterpret_cast<const float4*>(pr - N)) : p4;
        pz4 = gk > 0 ? __ldg(reinterpret_cast<const float4*>(pr - (size_t)N * N)) : p4;
        pm = gi0 > 0 ? __ldg(pr - 1) : p4.x;
    }
    const float* xr = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + 4 + ii;
    const float4 c4 = ld4(xr), ym4 = ld4(xr - XSW), zm4 = ld4(xr - (TJ + 2) * XSW);
    const float xm = xr[-1], xq = xr[4];
    const float xc[4] = {c4.x, c4.y, c4.z, c4.w};
    const float xl[4] = {xm, c4.x, c4.y, c4.z}, xn[4] = {c4.y, c4.z, c4.w, xq};
    const float ym[4] = {ym4.x, ym4.y, ym4.z, ym4.w}, zm[4] = {zm4.x, zm4.y, zm4.z, zm4.w};
    const float4 g4 = ld4(lbuf + gi0);
    const float gg[4] = {g4.x, g4.y, g4.z, g4.w};
    const float av[4] = {a4.x, a4.y, a4.z, a4.w};
    float tvg[4] = {0.f, 0.f, 0.f, 0.f};
    float d1[4], d2[4], d3[4], gn[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        d1[c] = (gi0 + c) > 0 ? xc[c] - xl[c] : 0.f;
        d2[c] = gj > 0 ? xc[c] - ym[c] : 0.f;
        d3[c] = gk > 0 ? xc[c] - zm[c] : 0.f;
        gn[c] = sqrt_(d1[c] * d1[c] + d2[c] * d2[c] + d3[c] * d3[c]);
    }
    if (has_beta) {
        const float* sr = SS + (kk * (TJ + 1) + jj) * SSW + ii;
        const float4 s4 = ld4(sr), sy4 = ld4(sr + SSW), sz4 = ld4(sr + (TJ + 1) * SSW);
        const float sq = sr[4];
        const float4 yp4 = ld4(xr + XSW), zp4 = ld4(xr + (TJ + 2) * XSW);
        const float s0[4] = {s4.x, s4.y, s4.z, s4.w}, sx[4] = {s4.y, s4.z, s4.w, sq};
        const float sy[4] = {sy4.x, sy4.y, sy4.z, sy4.w}, sz[4] = {sz4.x, sz4.y, sz4.z, sz4.w};
        const float yp[4] = {yp4.x, yp4.y, yp4.z, yp4.w}, zp[4] = {zp4.x, zp4.y, zp4.z, zp4.w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float t = s0[c] * (d1[c] + d2[c] + d3[c]);
            if (gi0 + c < N - 1) t -= sx[c] * (xn[c] - xc[c]);
            if (gj < N - 1) t -= sy[c] * (yp[c] - xc[c]);
            if (gk < N - 1) t -= sz[c] * (zp[c] - xc[c]);
            tvg[c] = t;
        }
    }
    float wl1[4] = {1.f, 1.f, 1.f, 1.f}, wtv[4] = {1.f, 1.f, 1.f, 1.f};
    if (!p.convex) {
        float ws[4] = {xc[0], xc[1], xc[2], xc[3]};
        if (p.wl1src) {
            if (p.wl1src == p.anchor) {
#pragma unroll
                for (int c = 0; c < 4; ++c) ws[c] = av[c];
            } else {
                const float4 w4 = __ldg(reinterpret_cast<const float4*>(p.wl1src + gidx));
                ws[0] = w4.x; ws[1] = w4.y; ws[2] = w4.z; ws[3] = w4.w;
            }
        }
        if (p.wtvf) {
            const float4 w4 = __ldg(reinterpret_cast<const float4*>(p.wtvf + gidx));
            wtv[0] = w4.x; wtv[1] = w4.y; wtv[2] = w4.z; wtv[3] = w4.w;
        } else {
#pragma unroll
            for (int c = 0; c < 4; ++c) wtv[c] = rcp_(gn[c] + epsp);
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) wl1[c] = rcp_(fabsf(ws[c]) + eps);
    }
    float base[4] = {xc[0], xc[1], xc[2], xc[3]};
    if (p.fista) {
        const float4 o4 = __ldg(reinterpret_cast<const float4*>(p.xold + gidx));
        base[0] = o4.x; base[1] = o4.y; base[2] = o4.z; base[3] = o4.w;
    }
    float nx[4], spec[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        // update + prox (regularizer.cpp:193-205, 103-110)
        float gs = 2.f * (gg[c] * invL) + 2.f * gamma * (xc[c] - av[c]);
        if (has_beta) gs += beta * tvg[c];
        float v = xc[c] - lr * gs;
        if (has_alpha) {
            const float th = lr * alpha * wl1[c];
            v = fabsf(v) <= th ? 0.f : v - copysignf(th, v);
        }
        nx[c] = v;
        spec[c] = p.fista ? v + theta * (v - base[c]) : v;
        const float dx = v - base[c];
        fa[9] += dx * dx;
        fa[10] += v * v;
    }
    *reinterpret_cast<float4*>(p.xnext + gidx) = make_float4(nx[0], nx[1], nx[2], nx[3]);
    if (p.fista)
        *reinterpret_cast<float4*>(p.ynext + gidx) = make_float4(spec[0], spec[1], spec[2], spec[3]);
    st4(lbuf + gi0, spec[0], spec[1], spec[2], spec[3]);
    if (p.audit) {
        float pl1[4], ptv[4];
        if (p.xprev) {
            const float pc[4] = {p4.x, p4.y, p4.z, p4.w}, pl[4] = {pm, p4.x, p4.y, p4.z};
            const float py[4] = {py4.x, py4.y, py4.z, py4.w}, pz[4] = {pz4.x, pz4.y, pz4.z, pz4.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float e1 = pc[c] - pl[c];
                const float e2 = pc[c] - py[c];
                const float e3 = pc[c] - pz[c];
                pl1[c] = rcp_(fabsf(pc[c]) + eps);
                ptv[c] = rcp_(sqrt_(e1 * e1 + e2 * e2 + e3 * e3) + epsp);
            }
        }
        const float inv2mu = 0.5f * rcp_(mu);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float ax = fabsf(xc[c]);
            const float g = gn[c];
            const float hb = g < mu ? g * g * inv2mu : g - 0.5f * mu;
            fa[0] += wl1[c] * ax;
            fa[1] += wtv[c] * hb;
            fa[2] += wtv[c] * g;
            fa[3] += __logf(ax + eps);
            fa[4] += __logf(g + epsp);
            const float dd = xc[c] - av[c];
            fa[5] += dd * dd;
            if (p.xprev) {
                fa[6] += pl1[c] * ax;
                fa[7] += ptv[c] * hb;
                fa[8] += ptv[c] * g;
            }
        }
    }
}

template <typename R, int N>
__global__ void __launch_bounds__(SwGeo<R, N>::NT, SwGeo<R, N>::MINB)
sweep_kernel(SweepParams<R> p, const __grid_constant__ CUtensorMap tmx,
             const __grid_constant__ CUtensorMap tmg) {
    using G = SwGeo<R, N>;
    using C = Cx<R>;
    constexpr int Nh = G::Nh, E = G::EX, T = G::TX, TJ = G::TJ, TK = G::TK, LPC = G::LPC;
    constexpr int CI = G::CI, PADX = G::PADX, NT = G::NT, NW = G::NW;
    constexpr int XSW = G::XSW, XPW = G::XPW, SSW = G::SSW;
    if (p.st && ld_done(p.st)) return;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* lines = reinterpret_cast<C*>(smem_raw + G::OFF_LINES);   // [LPCB][PADX]
    R* XS0 = reinterpret_cast<R*>(smem_raw + G::OFF_XS);        // [2][TK+2][TJ+2][XSW]
    R* XP = reinterpret_cast<R*>(smem_raw + G::OFF_XP);         // [TK+1][TJ+1][XPW]
    R* SS = reinterpret_cast<R*>(smem_raw + G::OFF_SS);         // [TK+1][TJ+1][SSW]
    C* Gs = reinterpret_cast<C*>(smem_raw + G::OFF_G);          // TMA-staged spectrum rows
    double* red = reinterpret_cast<double*>(smem_raw + G::OFF_RED);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);  // x box [2], rows
    stage_table(tw, p.twN, N);

    const int tid = threadIdx.x;
    const int lane = tid & 31, wid = tid >> 5;
    // FFT-phase mapping: line group lg (T threads), position t
    // every thread runs the FFT code (warp-synchronous); groups past the tile's
    // LPC lines work on scratch buffers and touch no global memory
    const int lg = tid / T, t = tid % T;
    const bool fft_active = lg < LPC;
    C* buf = lines + lg * PADX;
    R* rl = reinterpret_cast<R*>(buf);
    const PadAddr pad{};
    const WarpSync wsync{};

    const R eps = R(p.eps), epsp = R(p.eps_prime), mu = R(p.mu);
    const R lr = R(p.lr), alpha = R(p.alpha), beta = R(p.beta), gamma = R(p.gamma);
    const R invL = R(p.invL);
    const bool has_beta = p.beta > 0.0, has_alpha = p.alpha > 0.0;
    const R theta = (p.fista && p.st) ? R(p.theta[p.st->iter]) : R(0);

    double acc[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) acc[q] = 0.0;

    // TMA issue helpers (one elected thread); step = (tile, chunk) of this CTA
    auto issue_x = [&](int tile_, int chunk_, int b) {
        const int tj0 = (tile_ % (N / TJ)) * TJ, tk0 = (tile_ / (N / TJ)) * TK;
        mbar_expect_tx(&bar[b], G::XBOX_BYTES);
        tma_load_3d(reinterpret_cast<unsigned char*>(XS0) + b * G::XS_BYTES, &tmx,
                    chunk_ * CI - 4, tj0 - 1, tk0 - 1, &bar[b]);
    };
    auto issue_g = [&](int tile_) {
        const int tj0 = (tile_ % (N / TJ)) * TJ, tk0 = (tile_ / (N / TJ)) * TK;
        mbar_expect_tx(&bar[2], G::GBYTES);
        for (int kk = 0; kk < TK; ++kk)
            for (int hb = 0; hb < G::NHB; ++hb)
                tma_load_2d(Gs + (kk * G::NHB + hb) * TJ * G::GW, &tmg, hb * G::GW,
                            (tk0 + kk) * N + tj0, &bar[2]);
    };
    if constexpr (G::V4) {
        if (tid == 0) {
            mbar_init(&bar[0], 1);
            mbar_init(&bar[1], 1);
            mbar_init(&bar[2], 1);
            mbar_fence_init();
        }
        __syncthreads();
        if (tid == 0 && blockIdx.x < G::NTILES) {
            issue_g(blockIdx.x);
            issue_x(blockIdx.x, 0, 0);
        }
    }
    __syncthreads();

    int q_tile = 0;
    for (int tile = blockIdx.x; tile < G::NTILES; tile += gridDim.x, ++q_tile) {
        const int j0 = (tile % (N / TJ)) * TJ;
        const int k0 = (tile / (N / TJ)) * TK;
        // line lg of the tile: (kk, jj) = (lg / TJ, lg % TJ)
        const int my_j = j0 + (lg % TJ), my_k = k0 + (lg / TJ);
        C* Srow = p.S + ((size_t)my_k * N + my_j) * Nh;

        // ---- 1. C2R: G rows -> g (unnormalised) in the line buffers ------------
        if (!(p.dbg & 1)) {
            C v[E];
            if constexpr (G::V4) {
                mbar_wait(&bar[2], q_tile & 1);
                const int kk = lg / TJ, jj = lg % TJ;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = t + T * m;
                    v[m] = fft_active
                               ? Gs[((kk * G::NHB + hh / G::GW) * TJ + jj) * G::GW + hh % G::GW]
                               : cx<C>(R(0), R(0));
                }
            } else {
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = fft_active ? Srow[t + T * m] : cx<C>(R(0), R(0));
            }
#pragma unroll
            for (int m = 0; m < E; ++m) buf[pad(t + T * m)] = v[m];
            __syncwarp();
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int hh = t + T * m;
                const C q = v[m];
                if (hh == 0) {
                    v[m] = cx<C>(q.x + q.y, q.x - q.y);
                } else {
                    const C qm = buf[pad(Nh - hh)];
                    const C a = cx<C>(q.x + qm.x, q.y - qm.y);
                    const C d = cx<C>(q.x - qm.x, q.y + qm.y);
                    const C bb = cmulc(d, tw[hh]);
                    v[m] = cx<C>(a.x - bb.y, a.y + bb.x);
                }
            }
            __syncwarp();
            fft_regs<Nh, E, N, false>(v, t, buf, pad, tw, wsync);
            __syncwarp();
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int pp = t + T * m;
                rl[2 * pp] = v[m].x;
                rl[2 * pp + 1] = v[m].y;
            }
        }
        __syncthreads();
        if constexpr (G::V4) {  // the staged rows are consumed: prefetch the next tile's
            if (tid == 0 && tile + (int)gridDim.x < G::NTILES) issue_g(tile + gridDim.x);
        }

        // ---- 2. sweep in chunks along x -------------------------------------------
        // per-tile partials in R (fp32 in product mode: N/32 * LPC/NW terms per
        // thread), folded into the fp64 totals once per tile
        R fa[NP1];
#pragma unroll
        for (int q = 0; q < NP1; ++q) fa[q] = R(0);
        for (int ci = 0; ci < G::NCH; ++ci) {
            const int i0 = ci * CI;
            const int step = q_tile * G::NCH + ci;
            R* XS = XS0 + (G::V4 ? (step & 1) * G::XSR * XSW : 0);
            if constexpr (G::V4) {
                // prefetch the next step's box into the other buffer (its readers
                // passed the barrier that ended the previous step), then wait
                if (tid == 0) {
                    if (ci + 1 < G::NCH) issue_x(tile, ci + 1, (step + 1) & 1);
                    else if (tile + (int)gridDim.x < G::NTILES)
                        issue_x(tile + gridDim.x, 0, (step + 1) & 1);
                }
                mbar_wait(&bar[step & 1], (step >> 1) & 1);
            } else {
                // stage x: rows (kk', jj') in [-1, TK] x [-1, TJ], global i in [i0-1, i0+CI]
                stage_rows<R, N, CI, TJ + 2>(XS, G::XSR, p.xcur, k0, j0, i0, true, wid, lane);
            }
            // x_prev: rows [-1, TK-1] x [-1, TJ-1], global i in [i0-1, i0+CI-1]
            if (!G::V4 && p.xprev)
                stage_rows<R, N, CI, TJ + 1>(XP, G::XPR, p.xprev, k0, j0, i0, false, wid, lane);
            __syncthreads();
            // s on the box (kk, jj, ii) in [0, TK] x [0, TJ] x [0, CI]: warp per row
            if constexpr (G::V4) {
                if (has_beta && !(p.dbg & 8)) sbox_v4<N, TJ>(SS, XS, p.wtvf, p.convex, k0, j0, i0, mu, epsp, wid, lane);
            } else {
            if (has_beta) {
                for (int r = wid; r < G::SSR; r += NW) {
                    const int kk = r / (TJ + 1), jj = r - kk * (TJ + 1);
                    const int gj = j0 + jj, gk = k0 + kk;
                    const bool rok = gj < N && gk < N;
                    const R* xrow = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + 4;
                    const R* wrow = p.wtvf ? p.wtvf + ((size_t)(rok ? gk : 0) * N + (rok ? gj : 0)) * N
                                           : nullptr;
                    R* srow = SS + r * SSW;
                    for (int ii = lane; ii <= CI; ii += 32) {
                        const int gi = i0 + ii;
                        R sv = R(0);
                        if (rok && gi < N) {
                            const R* xr = xrow + ii;
                            const R xc = xr[0];
                            const R d1 = gi > 0 ? xc - xr[-1] : R(0);
                            const R d2 = gj > 0 ? xc - xr[-XSW] : R(0);
                            const R d3 = gk > 0 ? xc - xr[-(TJ + 2) * XSW] : R(0);
                            const R gn = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                            R wt = R(1);
                            if (!p.convex) wt = wrow ? __ldg(wrow + gi) : rcp_(gn + epsp);
                            sv = wt * rcp_(mu > gn ? mu : gn);
                        }
                        srow[ii] = sv;
                    }
                }
            }
            }
            __syncthreads();
            // voxels: warp w -> lines w, w+NW, ...; lane -> x
            if constexpr (G::V4) {
                if (!(p.dbg & 16))
                for (int l = wid; l < LPC; l += NW)
                    voxels_v4<N, TJ>(p, fa, XS, XP, SS, reinterpret_cast<float*>(lines + l * PADX),
                                     k0 + l / TJ, j0 + l % TJ, l / TJ, l % TJ, i0, lane, has_alpha,
                                     has_beta, theta);
            } else {
            for (int l = wid; l < LPC; l += NW) {
                const int kk = l / TJ, jj = l % TJ;
                const int gk = k0 + kk, gj = j0 + jj;
                R* lbuf = reinterpret_cast<R*>(lines + l * PADX);
                const size_t rowoff = ((size_t)gk * N + gj) * N;
                for (int ii = lane; ii < CI; ii += 32) {
                    const int gi = i0 + ii;
                    const size_t gidx = rowoff + gi;
                    const R* xr = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + 4 + ii;
                    const R xc = xr[0];
                    const R d1 = gi > 0 ? xc - xr[-1] : R(0);
                    const R d2 = gj > 0 ? xc - xr[-XSW] : R(0);
                    const R d3 = gk > 0 ? xc - xr[-(TJ + 2) * XSW] : R(0);
                    const R gn = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                    const R av = __ldg(p.anchor + gidx);
                    R wl1 = R(1), wtv = R(1);
                    if (!p.convex) {
                        const R wsv = p.wl1src ? (p.wl1src == p.anchor ? av : __ldg(p.wl1src + gidx))
                                               : xc;
                        wl1 = rcp_(fabs(wsv) + eps);
                        wtv = p.wtvf ? __ldg(p.wtvf + gidx) : rcp_(gn + epsp);
                    }
                    R tvg = R(0);
                    if (has_beta) {
                        const R* sr = SS + (kk * (TJ + 1) + jj) * SSW + ii;
                        tvg = sr[0] * (d1 + d2 + d3);
                        if (gi < N - 1) tvg -= sr[1] * (xr[1] - xc);
                        if (gj < N - 1) tvg -= sr[SSW] * (xr[XSW] - xc);
                        if (gk < N - 1) tvg -= sr[(TJ + 1) * SSW] * (xr[(TJ + 2) * XSW] - xc);
                    }
                    // update + prox (regularizer.cpp:193-205, 103-110)
                    const R g = lbuf[gi] * invL;
                    R gs = R(2) * g + R(2) * gamma * (xc - av);
                    if (has_beta) gs += beta * tvg;
                    R nx = xc - lr * gs;
                    if (has_alpha) {
                        const R th = lr * alpha * wl1;
                        nx = fabs(nx) <= th ? R(0) : nx - copysign(th, nx);
                    }
                    R base = xc;
                    if (p.fista) base = __ldg(p.xold + gidx);
                    p.xnext[gidx] = nx;
                    R spec = nx;
                    if (p.fista) {
                        spec = nx + theta * (nx - base);
                        p.ynext[gidx] = spec;
                    }
                    lbuf[gi] = spec;
                    if (p.audit) {
                        const R ax = fabs(xc);
                        const R hb = gn < mu ? gn * gn / (R(2) * mu) : gn - mu / R(2);
                        fa[0] += R(wl1 * ax);
                        fa[1] += R(wtv * hb);
                        fa[2] += R(wtv * gn);
                        fa[3] += R(log_(ax + eps));
                        fa[4] += R(log_(gn + epsp));
                        const R dd = xc - av;
                        fa[5] += R(dd * dd);
                        if (p.xprev) {
                            const R* pr = XP + ((kk + 1) * (TJ + 1) + (jj + 1)) * XPW + 4 + ii;
                            const R pc = pr[0];
                            const R e1 = gi > 0 ? pc - pr[-1] : R(0);
                            const R e2 = gj > 0 ? pc - pr[-XPW] : R(0);
                            const R e3 = gk > 0 ? pc - pr[-(TJ + 1) * XPW] : R(0);
                            const R pl1 = rcp_(fabs(pc) + eps);
                            const R ptv = rcp_(sqrt_(e1 * e1 + e2 * e2 + e3 * e3) + epsp);
                            fa[6] += R(pl1 * ax);
                            fa[7] += R(ptv * hb);
                            fa[8] += R(ptv * gn);
                        }
                    }
                    const R dx = nx - base;
                    fa[9] += R(dx * dx);
                    fa[10] += R(nx * nx);
                }
            }
            }
            __syncthreads();
        }
#pragma unroll
        for (int q = 0; q < NP1; ++q) acc[q] += (double)fa[q];

        // ---- 3. R2C of the new iterate (line buffers) -> spectrum rows -------------
        if (!(p.dbg & 2)) {
            C v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int pp = t + T * m;
                v[m] = cx<C>(rl[2 * pp], rl[2 * pp + 1]);
            }
            __syncwarp();
            fft_regs<Nh, E, N, true>(v, t, buf, pad, tw, wsync);
            __syncwarp();
#pragma unroll
            for (int m = 0; m < E; ++m) buf[pad(t + T * m)] = v[m];
            __syncwarp();
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int hh = t + T * m;
                const C z = v[m];
                C out;
                if (hh == 0) {
                    out = cx<C>(z.x + z.y, z.x - z.y);
                } else {
                    const C zm = buf[pad(Nh - hh)];
                    const C e = cx<C>(R(0.5) * (z.x + zm.x), R(0.5) * (z.y - zm.y));
                    const C o = cx<C>(R(0.5) * (z.y + zm.y), R(-0.5) * (z.x - zm.x));
                    out = cadd(e, cmul(o, tw[hh]));
                }
                if (fft_active) Srow[hh] = out;
            }
        }
        __syncthreads();
    }

    if (p.part) {
        block_sum<NP1>(acc, red);
        if (threadIdx.x == 0)
#pragma unroll
            for (int q = 0; q < NP1; ++q) p.part[(size_t)blockIdx.x * NP1 + q] = acc[q];
    }
}

} // namespace cm
