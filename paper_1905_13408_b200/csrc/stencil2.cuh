// K1 (fp32 and fp64, N >= 128, N % 8 == 0) — z-marching register-blocked stencil sweep.
//
// Same mathematics as stencil.cuh (regularizer.cpp:44-59, 72-85, 103-110,
// 125-149, 193-205; gradient.cpp:7-64), reorganised so that every TV dual scale
//     s(q) = w_tv(q) / max(mu, |Dx(q)|) = 1 / ((|Dx(q)| + eps') max(mu, |Dx(q)|))
// is computed exactly once and every input sample is read from shared memory
// once per use:
//   * a CTA owns a CI = 32 VW (x) by TJ (y) column of voxels and marches along z over
//     KC planes; warp w owns row j0 + w, lane l owns x = i0 + VW l .. VW l + VW-1 (VW = 4
//     in fp32, 2 in the fp64 parity mode); one
//     extra warp computes s on the forward halo row j0 + TJ;
//   * per plane q, TMA brings the x slab (rows j0-1 .. j0+TJ, x halo +-1), the
//     x_{i-1} slab (rows j0-1 .. j0+TJ-1), and the g and anchor rows into a
//     4-deep ring (prefetch distance 2 planes, mbarrier complete_tx);
//   * step k: s(., k+1) is computed from the plane k+1 slab and the rolling
//     x(., k), published in a 3-deep shared ring, one barrier; then voxel (j, k)
//     uses s(j,k) and s(j,k+1) from registers, s(j+1,k) from shared memory and
//     s(i+1) / x(i+-1) from shuffles.
#pragma once

#include "cm_common.cuh"
#include "kernels.cuh"
#include "stencil.cuh"
#include "tma.cuh"

#include <utility>

#ifndef CM_S2_MINB
#define CM_S2_MINB 4
#endif
#ifndef CM_S2_PD
#define CM_S2_PD 2  // TMA prefetch distance in planes (2 or 3; the ring has 4 slots)
#endif
#ifndef CM_S2_MINB_D
#define CM_S2_MINB_D 3  // fp64: 136 registers (double accumulators and parameters)
#endif
#ifndef CM_S2_TJ
#define CM_S2_TJ 4  // rows per CTA (+1 halo-row warp); 4 CTAs per SM (8: 2 CTAs, 3.5% slower)
#endif
#ifndef CM_S2_TJ_D
#define CM_S2_TJ_D 4  // fp64 rows per CTA
#endif

namespace cm {

// planes per march: the KC in {64, 32, 16, 8} minimising the plane steps of the
// busiest CTA slot (148 SMs x CM_S2_MINB), ceil(tiles / slots) x (KC + 2 for the
// march prologue); ties keep the longer march. 512^3 / 384^3 / 256^3: 64; 128^3:
// 8 (64-plane marches ran 64 CTAs for the whole sweep: 57 -> 19 us)
__host__ __device__ constexpr int s2_kc(int n, int ci = 128, int minb = CM_S2_MINB, int tj = CM_S2_TJ) {
    if (n < 64) return n;
    int best = 64;
    long best_cost = -1;
    for (int kc = 64; kc >= 8; kc /= 2) {
        if (n % kc) continue;
        const long tiles = (long)((n + ci - 1) / ci) * (n / tj) * (n / kc);
        const long slots = 148L * minb;
        const long cost = (tiles + slots - 1) / slots * (kc + 2);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = kc;
        }
    }
    return best;
}

// real-type overloads (no implicit float -> double promotion in the fp32 sweep)
__device__ __forceinline__ float s2abs(float v) { return fabsf(v); }
__device__ __forceinline__ double s2abs(double v) { return fabs(v); }
__device__ __forceinline__ float s2min(float a, float b) { return fminf(a, b); }
// fp64: compare-and-select (fmin / fmax carry NaN handling; operands here are finite)
__device__ __forceinline__ double s2min(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ float s2max(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double s2max(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ float s2fma(float a, float b, float c) { return fmaf(a, b, c); }
__device__ __forceinline__ double s2fma(double a, double b, double c) { return fma(a, b, c); }
// reciprocal of an operand known positive and normal here ((|x| + eps)(|Dx| + eps'),
// (|Dx| cg + ce) max(mu, |Dx|), max(mu, |Dx|): eps, eps', mu > 0 are validated):
// fp64 skips rcp_'s 1/0 guard
__device__ __forceinline__ float s2rcp(float v) { return rcp_(v); }
__device__ __forceinline__ double s2rcp(double v) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
    double e = fma(-v, y, 1.0);
    double z = fma(y, fma(e, e, e), y);
    e = fma(-v, z, 1.0);
    return fma(z, e, z);
}

// R = float: 4 voxels (one float4) per lane, 128-wide x tiles; R = double (the
// fp64 parity mode): 2 voxels (one double2) per lane, 64-wide x tiles
template <typename R, int N> struct S2GeoT {
    static constexpr int VW = 16 / (int)sizeof(R);  // voxels per lane
    static constexpr int CI = 32 * VW;
    static constexpr int MINB = sizeof(R) == 4 ? CM_S2_MINB : CM_S2_MINB_D;
    static constexpr int TJ = sizeof(R) == 4 ? CM_S2_TJ : CM_S2_TJ_D;
    static constexpr int KC = s2_kc(N, CI, MINB, TJ);  // planes per march
    static constexpr int NW = TJ + 1;            // + halo-row warp
    static constexpr int NT = NW * 32;
    static constexpr int XW = CI + 2 * VW;       // slab row: global i0-VW .. i0+CI+VW-1
    static constexpr int XR = TJ + 2;            // x rows j0-1 .. j0+TJ
    static constexpr int PR = TJ + 1;            // x_prev rows j0-1 .. j0+TJ-1
    static constexpr int GR = TJ;                // g / anchor rows j0 .. j0+TJ-1
    static constexpr uint32_t XB = XR * XW * sizeof(R), PB = PR * XW * sizeof(R), GB = GR * CI * sizeof(R);
    static constexpr size_t al(size_t v) { return (v + 127) / 128 * 128; }
    static constexpr size_t OFF_P = al(XB), OFF_G = al(OFF_P + PB), OFF_A = al(OFF_G + GB);
    static constexpr size_t STAGE = al(OFF_A + GB);
    static constexpr int NSTAGE = 4;
    static constexpr int SW = CI + VW;           // s row (+ halo column at CI)
    static constexpr size_t OFF_S = NSTAGE * STAGE;
    static constexpr size_t SROW3 = (size_t)(TJ + 1) * SW;   // floats per s ring slot
    static constexpr size_t S_BYTES = 3 * SROW3 * sizeof(R);
    static constexpr size_t OFF_RED = al(OFF_S + S_BYTES);
    static constexpr size_t OFF_BAR = OFF_RED + 32 * NP1 * 8;
    static constexpr size_t SMEM = OFF_BAR + NSTAGE * 8;
    static constexpr int NTI = (N + CI - 1) / CI, NTJ = N / TJ, NTK = N / KC;  // last x tile partial
    static constexpr int NTILES = NTI * NTJ * NTK;  // single GPU (nk = N)
};
template <int N> using S2Geo = S2GeoT<float, N>;

#ifdef CM_S2_MAXREG
#define CM_S2_BOUNDS __maxnreg__(CM_S2_MAXREG)
#else
#define CM_S2_BOUNDS __launch_bounds__(S2GeoT<R, N>::NT, S2GeoT<R, N>::MINB)
#endif

// compile-time mode of a sweep: dead terms, branches and accumulators vanish
enum S2Flags { S2_AUDIT = 1, S2_PREV = 2, S2_TRACE = 4, S2_STEP = 8, S2_FISTA = 16 };

// partial-sum slots a mode produces (kernels.cuh NP1 layout)
__host__ __device__ constexpr unsigned s2_used(int F) {
    return ((F & S2_AUDIT) ? (1u | 2u | 32u | ((F & S2_PREV) ? 64u | 128u : 0u) |
                              ((F & S2_TRACE) ? 4u | 8u | 16u | ((F & S2_PREV) ? 256u : 0u) : 0u))
                           : 0u) |
           ((F & S2_STEP) ? 512u | 1024u : 0u) | ((F & S2_FISTA) ? 2048u : 0u);
}

template <typename R, int N, int F>
__global__ void CM_S2_BOUNDS
stencil2_kernel(StencilParams<R> p, const __grid_constant__ CUtensorMap tmx,
                const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmg,
                const __grid_constant__ CUtensorMap tma) {
    using G = S2GeoT<R, N>;
    using V = Vec16<R>;
    constexpr int VW = G::VW;
    constexpr bool AUDIT = F & S2_AUDIT, PREV = AUDIT && (F & S2_PREV);
    constexpr bool TRACE = AUDIT && (F & S2_TRACE), STEP = F & S2_STEP, FISTA = F & S2_FISTA;
    constexpr unsigned USED = s2_used(F);
    constexpr int CI = G::CI, TJ = G::TJ, KC = G::KC, XW = G::XW, SW = G::SW;
    pdl_trigger();
    pdl_wait();
    if (p.st && ld_done(p.st)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    R* Sring = reinterpret_cast<R*>(smem_raw + G::OFF_S);   // [3][TJ+1][SW]
    double* red = reinterpret_cast<double*>(smem_raw + G::OFF_RED);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);
    const uint32_t smem_s = smem_u32(smem_raw), bar_s = smem_s + (uint32_t)G::OFF_BAR;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;  // w = row within tile, TJ = halo
    const bool halo = (w == TJ);
    // fp32 parameters as references into the (constant-bank) kernel parameters
    const R &eps = p.f_eps, &epsp = p.f_epsp, &mu = p.f_mu, &lr = p.f_lr, &lra = p.f_lra;
    const R &beta = p.f_beta, &g2 = p.f_g2, &inv2mu = p.f_inv2mu, &hmu = p.f_hmu;
    const R &cg = p.f_cg, &ce = p.f_ce;
    const bool has_beta = p.beta > 0.0, has_alpha = p.alpha > 0.0;
    constexpr bool with_prev = PREV;
    const bool convex = p.convex != 0;
    // s = 1/((g cg + ce) max(mu, g)): (cg, ce) = (1, eps') reweighted, (0, 1) convex
    const R theta = (FISTA && p.st) ? R(p.theta[p.st->iter - p.st->mom_base]) : R(0);

    if (tid == 0) {
        for (int q = 0; q < G::NSTAGE; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    // per-warp fp64 partial sums of the CTA's tiles (no fp64 registers held)
    for (int q = tid; q < 32 * NP1; q += blockDim.x) red[q] = 0.0;
    __syncthreads();

    // partials in R: fa over 8 planes, fb over the tile, then fp64 per warp
    R fa[NP1], fb[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) fa[q] = fb[q] = R(0);

    uint32_t phase_bits = 0;  // parity of the next wait on each ring slot
    const int koff = p.koff, zs = p.zshift;
    const int ntiles = G::NTI * G::NTJ * (p.nk / KC);
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int i0 = (tile % G::NTI) * CI;
        const int j0 = ((tile / G::NTI) % G::NTJ) * TJ;
        const int k0 = (tile / (G::NTI * G::NTJ)) * KC;
        // plane q (k0-1 .. k0+KC) lives in ring slot (q - k0 + 1) % NSTAGE
        auto slot_of = [&](int q) { return (q - k0 + 1) & (G::NSTAGE - 1); };
        auto stage = [&](int q) { return smem_raw + (size_t)slot_of(q) * G::STAGE; };
        auto issue = [&](int q) {  // q: local plane (ghost planes at -1 and nk)
            if (q > k0 + KC) return;
            const int sl = slot_of(q);
            const uint32_t bs = bar_s + 8u * sl, ss = smem_s + (uint32_t)((size_t)sl * G::STAGE);
            mbar_expect_tx_s(bs, G::XB + (with_prev ? G::PB : 0u) + 2 * G::GB);
            tma_load_3d_s(ss, &tmx, i0 - VW, j0 - 1, q + zs, bs);
            if (with_prev) tma_load_3d_s(ss + (uint32_t)G::OFF_P, &tmp, i0 - VW, j0 - 1, q + zs, bs);
            // g / anchor rows of planes past the march are never read; out of grid -> 0
            tma_load_3d_s(ss + (uint32_t)G::OFF_G, &tmg, i0, j0, q + zs, bs);
            tma_load_3d_s(ss + (uint32_t)G::OFF_A, &tma, i0, j0, q + zs, bs);
        };
        auto wait = [&](int q) {
            const int sl = slot_of(q);
            mbar_wait_s(bar_s + 8u * sl, (phase_bits >> sl) & 1u);
            phase_bits ^= (1u << sl);
        };
        if (tid == 0) {
            issue(k0 - 1);
            issue(k0);
            issue(k0 + 1);
            if (CM_S2_PD == 3) issue(k0 + 2);
        }
        wait(k0 - 1);
        wait(k0);

        const int gj = j0 + w;                 // this warp's row (halo warp: j0 + TJ)
        const int ii = VW * lane;
        const int gi0 = i0 + ii;
        const bool row_in = gj < N;
        // partial last x tile (N % CI != 0): the lane's VW voxels are all in or
        // all out; out-of-grid lanes keep s = 0 and join the shuffles, but load,
        // store and accumulate nothing
        const bool col_in = gi0 < N;
        // replicate boundary (gradient.cpp:7-24): the backward neighbour of the
        // first row / column / plane is the voxel itself, so D = 0 there without
        // a per-voxel test; forward terms vanish because s = 0 outside the grid
        const int ry = gj > 0 ? w : w + 1;     // slab row of j-1
        const bool xlo = (i0 == 0);
        // x slab row r (global j0 - 1 + r) of plane q, at this lane's 4 voxels
        auto xrow = [&](int q, int r) -> const R* {
            return reinterpret_cast<const R*>(stage(q)) + r * XW + VW + ii;
        };
        // s on row w of plane q from the slabs of q and q-1 (rows w+1, w in slab coords)
        // returns s[4], plus |Dx|, d-sum for the voxels; halo column (i0+CI) via lane 31
        auto s_row = [&](int q, R (&xq)[VW], R (&sv)[VW], R (&gn)[VW], R (&ds)[VW]) {
            const R* xr = xrow(q, w + 1);
            const R* yr = xrow(q, ry);
            const R* zr = koff + q > 0 ? xrow(q - 1, w + 1) : xr;
            R yv[VW], zv[VW];
            V::ld(xr, xq);
            V::ld(yr, yv);
            V::ld(zr, zv);
            R xl = __shfl_up_sync(0xffffffffu, xq[VW - 1], 1);
            if (lane == 0) xl = xlo ? xq[0] : xr[-1];
            R xlv[VW];
            xlv[0] = xl;
#pragma unroll
            for (int c = 1; c < VW; ++c) xlv[c] = xq[c - 1];
            const bool qin = koff + q < N && row_in && col_in;
#pragma unroll
            for (int c = 0; c < VW; ++c) {
                const R d1 = xq[c] - xlv[c], d2 = xq[c] - yv[c], d3 = xq[c] - zv[c];
                const R g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                const R mx = mu > g ? mu : g;
                const R s = s2rcp(s2fma(g, cg, ce) * mx);  // convex: 1/mx
                sv[c] = qin ? s : R(0);
                gn[c] = g;
                ds[c] = d1 + d2 + d3;
            }
        };
        // s on the column x = i0 + CI of tile row `lane` (0 .. TJ): computed by the
        // halo-row warp, so the row warps carry no divergent halo-column work
        auto s_col = [&](int q) -> R {
            const int r = lane, gjr = j0 + lane;
            if (r > TJ || koff + q >= N || gjr >= N || i0 + CI >= N) return R(0);
            const R* xb = reinterpret_cast<const R*>(stage(q)) + VW + CI;
            const R* zb = koff + q > 0 ? reinterpret_cast<const R*>(stage(q - 1)) + VW + CI : xb;
            const R xc = xb[(r + 1) * XW];
            const R d1 = xc - xb[(r + 1) * XW - 1];
            const R d2 = xc - xb[(gjr > 0 ? r : r + 1) * XW];
            const R d3 = xc - zb[(r + 1) * XW];
            const R g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
            const R mx = mu > g ? mu : g;
            if (p.wtvf && !convex)
                return __ldg(p.wtvf + ((size_t)(q + zs) * N + gjr) * N + i0 + CI) * s2rcp(mx);
            return s2rcp(s2fma(g, cg, ce) * mx);
        };
        // per_m_step weights come from a frozen field: s uses w_tv from it
        auto apply_wtvf = [&](int q, R (&sv)[VW], R (&gn)[VW]) {
            if (!p.wtvf || convex || !(koff + q < N && row_in && col_in)) return;
            R wt[VW];
            V::ldg(p.wtvf + ((size_t)(q + zs) * N + gj) * N + gi0, wt);
#pragma unroll
            for (int c = 0; c < VW; ++c) {
                const R mx = mu > gn[c] ? mu : gn[c];
                sv[c] = wt[c] * s2rcp(mx);
            }
        };

        // ---- prologue: s(., k0), rolling state of plane k0 and x_prev(k0-1)
        R x_cur[VW], s_cur[VW], gn_cur[VW], ds_cur[VW];
        s_row(k0, x_cur, s_cur, gn_cur, ds_cur);
        apply_wtvf(k0, s_cur, gn_cur);
        // s ring: plane k in slot (k - k0) % 3, rotated by pointer
        R* Sc_ring = Sring;                        // slot of plane k
        R* Sn_ring = Sring + G::SROW3;             // slot of plane k + 1
        R* Sx_ring = Sring + 2 * G::SROW3;         // the third slot
        R* S0 = Sc_ring;
        if (has_beta) {
            V::st(S0 + w * SW + ii, s_cur);
            if (halo && lane <= TJ) S0[lane * SW + CI] = s_col(k0);
        }
        R xp_prev[VW];
#pragma unroll
        for (int c = 0; c < VW; ++c) xp_prev[c] = R(0);
        if (with_prev && !halo) {
            // plane k0-1 of x_prev (the plane itself at the global first plane)
            V::ld(reinterpret_cast<const R*>(stage(koff + k0 > 0 ? k0 - 1 : k0) + G::OFF_P) +
                      (w + 1) * XW + VW + ii,
                  xp_prev);
        }
        __syncthreads();

        // one plane of the march; the rolling state alternates between two
        // register sets (the loop is unrolled by two) instead of being copied
        R x_nb[VW], s_nb[VW], gn_nb[VW], ds_nb[VW];
        auto step = [&](int k, R (&x_cur)[VW], R (&s_cur)[VW], R (&gn_cur)[VW],
                        R (&ds_cur)[VW], R (&x_nx)[VW], R (&s_nx)[VW],
                        R (&gn_nx)[VW], R (&ds_nx)[VW]) {
            // prefetch distance 2: the slot of plane k-2 was released by the previous
            // barrier; distance 3 (CM_S2_PD=3): plane k+3 goes to the slot of k-1
            // after this step's barrier (all four slots in use, no more shared memory)
            if (CM_S2_PD == 2 && tid == 0) issue(k + 2);
            wait(k + 1);
            // ---- s of plane k+1 on this warp's row
            s_row(k + 1, x_nx, s_nx, gn_nx, ds_nx);
            apply_wtvf(k + 1, s_nx, gn_nx);
            R* Sn = Sn_ring;
            if (has_beta) {
                V::st(Sn + w * SW + ii, s_nx);
                if (halo && lane <= TJ) Sn[lane * SW + CI] = s_col(k + 1);
            }
            __syncthreads();
            if (CM_S2_PD == 3 && tid == 0) issue(k + 3);
            if (!halo && row_in) {
                // ---- voxel (j, k): update, prox, partials
                const R* Sc = Sc_ring;
                const size_t gidx = ((size_t)(k + zs) * N + gj) * N + gi0;
                const unsigned char* stk = stage(k);
                R gg[VW], av[VW];
                V::ld(reinterpret_cast<const R*>(stk + G::OFF_G) + w * CI + ii, gg);
                V::ld(reinterpret_cast<const R*>(stk + G::OFF_A) + w * CI + ii, av);
                R tvg[VW];
#pragma unroll
                for (int c = 0; c < VW; ++c) tvg[c] = R(0);
                if (has_beta) {
                    // x(j+1, k) and s(j+1, k): next row; x(i+1), s(i+1): next voxel
                    R yp[VW], sy[VW];
                    V::ld(xrow(k, w + 2), yp);
                    V::ld(Sc + (w + 1) * SW + ii, sy);
                    R xr4 = __shfl_down_sync(0xffffffffu, x_cur[0], 1);
                    R sr4 = __shfl_down_sync(0xffffffffu, s_cur[0], 1);
                    if (lane == 31) {
                        xr4 = xrow(k, w + 1)[VW];         // x at i0 + CI
                        sr4 = Sc[w * SW + CI];
                    }
                    R xn[VW], sxv[VW];
#pragma unroll
                    for (int c = 0; c + 1 < VW; ++c) {
                        xn[c] = x_cur[c + 1];
                        sxv[c] = s_cur[c + 1];
                    }
                    xn[VW - 1] = xr4;
                    sxv[VW - 1] = sr4;
#pragma unroll
                    for (int c = 0; c < VW; ++c)
                        tvg[c] = s_cur[c] * ds_cur[c] - sxv[c] * (xn[c] - x_cur[c]) -
                                 sy[c] * (yp[c] - x_cur[c]) - s_nx[c] * (x_nx[c] - x_cur[c]);
                }
                R wl1[VW], wtv[VW];
#pragma unroll
                for (int c = 0; c < VW; ++c) wl1[c] = wtv[c] = R(1);
                if (!convex) {
                    R ws[VW];
#pragma unroll
                    for (int c = 0; c < VW; ++c) ws[c] = x_cur[c];
                    if (p.wl1src) {
                        if (p.wl1src == p.anchor) {
#pragma unroll
                            for (int c = 0; c < VW; ++c) ws[c] = av[c];
                        } else if (col_in) {
                            V::ldg(p.wl1src + gidx, ws);
                        }
                    }
                    if (p.wtvf) {
                        if (col_in) V::ldg(p.wtvf + gidx, wtv);
#pragma unroll
                        for (int c = 0; c < VW; ++c) wl1[c] = s2rcp(s2abs(ws[c]) + eps);
                    } else {
#pragma unroll
                        for (int c = 0; c < VW; ++c) {
                            const R a = s2abs(ws[c]) + eps, b = gn_cur[c] + epsp;
                            const R r = s2rcp(a * b);
                            wl1[c] = b * r;
                            wtv[c] = a * r;
                        }
                    }
                }
                R base[VW];
#pragma unroll
                for (int c = 0; c < VW; ++c) base[c] = x_cur[c];
                if (FISTA && col_in) V::ldg(p.xold + gidx, base);
                R nx[VW];
#pragma unroll
                for (int c = 0; c < VW; ++c) {
                    R gs = R(2) * gg[c] + g2 * (x_cur[c] - av[c]);
                    if (has_beta) gs += beta * tvg[c];
                    R v = x_cur[c] - lr * gs;
                    if (has_alpha) {
                        const R th = lra * wl1[c];
                        // soft threshold, |v| <= th -> 0 (regularizer.cpp:107): v - clamp(v)
                        v = v - s2min(s2max(v, -th), th);
                    }
                    nx[c] = v;
                }
                if (!p.obj_only && col_in) V::st(p.xnext + gidx, nx);
                if (FISTA && !p.obj_only && col_in) {
                    R y[VW];
#pragma unroll
                    for (int c = 0; c < VW; ++c) y[c] = nx[c] + theta * (nx[c] - base[c]);
                    V::st(p.ynext + gidx, y);
                }
                if (FISTA && col_in) {
                    // restart test (O'Donoghue & Candes): (y_k - x_{k+1}) . (x_{k+1} - x_k)
#pragma unroll
                    for (int c = 0; c < VW; ++c) fa[11] += (x_cur[c] - nx[c]) * (nx[c] - base[c]);
                }
                if (STEP && col_in) {
#pragma unroll
                    for (int c = 0; c < VW; ++c) {
                        const R dx = nx[c] - base[c];
                        fa[9] += dx * dx;
                        fa[10] += nx[c] * nx[c];
                    }
                }
                if (AUDIT) {
                    R pl1[VW], ptv[VW];
#pragma unroll
                    for (int c = 0; c < VW; ++c) pl1[c] = ptv[c] = R(0);
                    if (with_prev) {
                        const R* P = reinterpret_cast<const R*>(stk + G::OFF_P);
                        R pc[VW], py[VW], pl[VW];
                        V::ld(P + (w + 1) * XW + VW + ii, pc);
                        V::ld(P + ry * XW + VW + ii, py);
                        R pm = __shfl_up_sync(0xffffffffu, pc[VW - 1], 1);
                        if (lane == 0) pm = xlo ? pc[0] : P[(w + 1) * XW + VW - 1];
                        pl[0] = pm;
#pragma unroll
                        for (int c = 1; c < VW; ++c) pl[c] = pc[c - 1];
#pragma unroll
                        for (int c = 0; c < VW; ++c) {
                            const R e1 = pc[c] - pl[c], e2 = pc[c] - py[c], e3 = pc[c] - xp_prev[c];
                            const R a = s2abs(pc[c]) + eps;
                            const R b = sqrt_(e1 * e1 + e2 * e2 + e3 * e3) + epsp;
                            const R r = s2rcp(a * b);
                            pl1[c] = b * r;
                            ptv[c] = a * r;
                            xp_prev[c] = pc[c];
                        }
                    }
#pragma unroll
                    for (int c = 0; c < VW; ++c) {
                        if (!col_in) break;
                        const R ax = s2abs(x_cur[c]), g = gn_cur[c];
                        const R hb = g < mu ? g * g * inv2mu : g - hmu;
                        fa[0] += wl1[c] * ax;
                        fa[1] += wtv[c] * hb;
                        const R dd = x_cur[c] - av[c];
                        fa[5] += dd * dd;
                        if (with_prev) {
                            fa[6] += pl1[c] * ax;
                            fa[7] += ptv[c] * hb;
                        }
                        if (TRACE) {
                            fa[2] += wtv[c] * g;
                            fa[3] += log_(ax + eps);
                            fa[4] += log_(g + epsp);
                            if (with_prev) fa[8] += ptv[c] * g;
                        }
                    }
                }
            }
            R* const sfree = Sc_ring;
            Sc_ring = Sn_ring;
            Sn_ring = Sx_ring;
            Sx_ring = sfree;
        };
        for (int k = k0; k < k0 + KC; k += 2) {
            step(k, x_cur, s_cur, gn_cur, ds_cur, x_nb, s_nb, gn_nb, ds_nb);
            step(k + 1, x_nb, s_nb, gn_nb, ds_nb, x_cur, s_cur, gn_cur, ds_cur);
            // fp32: flush the 8-plane partials into the tile partials (bounded
            // rounding); fp64 accumulates the tile in fa directly (fewer registers)
            if (sizeof(R) == 4 && USED && ((k + 1 - k0) & 7) == 7) {
#pragma unroll
                for (int q = 0; q < NP1; ++q)
                    if (USED & (1u << q)) {
                        fb[q] += fa[q];
                        fa[q] = R(0);
                    }
            }
        }
        // tile partials -> this warp's fp64 slots (lane order fixed: deterministic)
        if constexpr (USED != 0) {
#pragma unroll
            for (int q = 0; q < NP1; ++q)
                if (USED & (1u << q)) {
                    const double v = warp_sum(sizeof(R) == 4 ? (double)fb[q] : (double)fa[q]);
                    if (lane == 0) red[w * NP1 + q] += v;
                    fb[q] = R(0);
                    if (sizeof(R) == 8) fa[q] = R(0);
                }
        }
        // every issued plane (k0-1 .. k0+KC) has been waited on
        __syncthreads();
    }
    if (p.part && tid < NP1) {
        double t = 0.0;
        for (int v = 0; v < G::NW; ++v) t += red[v * NP1 + tid];
        p.part[(size_t)blockIdx.x * NP1 + tid] = t;
    }
}

// host: mode flags of a sweep and the matching instantiation
template <typename R> inline int s2_flags(const StencilParams<R>& p) {
    int f = 0;
    if (p.audit) {
        f |= S2_AUDIT;
        if (p.xprev) f |= S2_PREV;
        if (p.trace_full) f |= S2_TRACE;
    }
    if (p.steptol) f |= S2_STEP;
    if (p.fista) f |= S2_FISTA;
    return f;
}

#define CM_S2_MODES(X) X(0) X(8) X(1) X(9) X(3) X(11) X(5) X(13) X(7) X(15) X(16) X(24)

template <int N, typename R = float> inline cudaError_t stencil2_prepare() {
    cudaError_t e = cudaSuccess;
#define CM_S2_ATTR(FL)                                                                         \
    if (e == cudaSuccess)                                                                     \
        e = cudaFuncSetAttribute(stencil2_kernel<R, N, FL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)S2GeoT<R, N>::SMEM);
    CM_S2_MODES(CM_S2_ATTR)
#undef CM_S2_ATTR
    return e;
}

// launch with the programmatic-dependent-launch attribute (see pdl_wait)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(bool pdl, void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <int N, typename R>
inline cudaError_t stencil2_launch(StencilParams<R> p, int grid, cudaStream_t s,
                                   const CUtensorMap& tmx, const CUtensorMap& tmp,
                                   const CUtensorMap& tmg, const CUtensorMap& tma, bool pdl = false) {
    p.f_eps = R(p.eps);
    p.f_epsp = R(p.eps_prime);
    p.f_mu = R(p.mu);
    p.f_lr = R(p.lr);
    p.f_lra = R(p.lr * p.alpha);
    p.f_beta = R(p.beta);
    p.f_g2 = R(2.0 * p.gamma);
    p.f_inv2mu = R(0.5 / p.mu);
    p.f_hmu = R(0.5 * p.mu);
    p.f_cg = p.convex ? R(0) : R(1);
    p.f_ce = p.convex ? R(1) : R(p.eps_prime);
    switch (s2_flags(p)) {
#define CM_S2_CASE(FL)                                                                         \
    case FL:                                                                                   \
        return launch_pdl(pdl, stencil2_kernel<R, N, FL>, dim3(grid), dim3(S2GeoT<R, N>::NT),    \
                          S2GeoT<R, N>::SMEM, s, p, tmx, tmp, tmg, tma);
        CM_S2_MODES(CM_S2_CASE)
#undef CM_S2_CASE
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int N, typename R = float> inline cudaError_t stencil2_occupancy(int* occ) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stencil2_kernel<R, N, S2_AUDIT | S2_PREV>,
                                                         S2GeoT<R, N>::NT, S2GeoT<R, N>::SMEM);
}

} // namespace cm
