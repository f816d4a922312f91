// K1 (fp32, N % 128 == 0) — z-marching register-blocked stencil sweep.
//
// Same mathematics as stencil.cuh (regularizer.cpp:44-59, 72-85, 103-110,
// 125-149, 193-205; gradient.cpp:7-64), reorganised so that every TV dual scale
//     s(q) = w_tv(q) / max(mu, |Dx(q)|) = 1 / ((|Dx(q)| + eps') max(mu, |Dx(q)|))
// is computed exactly once and every input sample is read from shared memory
// once per use:
//   * a CTA owns a 128 (x) by TJ (y) column of voxels and marches along z over
//     KC planes; warp w owns row j0 + w, lane l owns x = i0 + 4l .. 4l+3; one
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
#ifndef CM_S2_TJ
#define CM_S2_TJ 4  // rows per CTA (+1 halo-row warp); 4 CTAs per SM (8: 2 CTAs, 3.5% slower)
#endif

namespace cm {

// planes per march: the KC in {64, 32, 16, 8} minimising the plane steps of the
// busiest CTA slot (148 SMs x CM_S2_MINB), ceil(tiles / slots) x (KC + 2 for the
// march prologue); ties keep the longer march. 512^3 / 384^3 / 256^3: 64; 128^3:
// 8 (64-plane marches ran 64 CTAs for the whole sweep: 57 -> 19 us)
__host__ __device__ constexpr int s2_kc(int n) {
    if (n < 64) return n;
    int best = 64;
    long best_cost = -1;
    for (int kc = 64; kc >= 8; kc /= 2) {
        if (n % kc) continue;
        const long tiles = (long)((n + 127) / 128) * (n / CM_S2_TJ) * (n / kc);
        const long slots = 148L * CM_S2_MINB;
        const long cost = (tiles + slots - 1) / slots * (kc + 2);
        if (best_cost < 0 || cost < best_cost) {
            best_cost = cost;
            best = kc;
        }
    }
    return best;
}

template <int N> struct S2Geo {
    static constexpr int CI = 128;
    static constexpr int TJ = CM_S2_TJ;
    static constexpr int KC = s2_kc(N);          // planes per march
    static constexpr int NW = TJ + 1;            // + halo-row warp
    static constexpr int NT = NW * 32;
    static constexpr int XW = 136;               // slab row: global i0-4 .. i0+131
    static constexpr int XR = TJ + 2;            // x rows j0-1 .. j0+TJ
    static constexpr int PR = TJ + 1;            // x_prev rows j0-1 .. j0+TJ-1
    static constexpr int GR = TJ;                // g / anchor rows j0 .. j0+TJ-1
    static constexpr uint32_t XB = XR * XW * 4, PB = PR * XW * 4, GB = GR * CI * 4;
    static constexpr size_t al(size_t v) { return (v + 127) / 128 * 128; }
    static constexpr size_t OFF_P = al(XB), OFF_G = al(OFF_P + PB), OFF_A = al(OFF_G + GB);
    static constexpr size_t STAGE = al(OFF_A + GB);
    static constexpr int NSTAGE = 4;
    static constexpr int SW = CI + 4;            // s row (+ halo column at CI)
    static constexpr size_t OFF_S = NSTAGE * STAGE;
    static constexpr size_t SROW3 = (size_t)(TJ + 1) * SW;   // floats per s ring slot
    static constexpr size_t S_BYTES = 3 * SROW3 * 4;
    static constexpr size_t OFF_RED = al(OFF_S + S_BYTES);
    static constexpr size_t OFF_BAR = OFF_RED + 32 * NP1 * 8;
    static constexpr size_t SMEM = OFF_BAR + NSTAGE * 8;
    static constexpr int NTI = (N + CI - 1) / CI, NTJ = N / TJ, NTK = N / KC;  // last x tile partial
    static constexpr int NTILES = NTI * NTJ * NTK;  // single GPU (nk = N)
};

#ifdef CM_S2_MAXREG
#define CM_S2_BOUNDS __maxnreg__(CM_S2_MAXREG)
#else
#define CM_S2_BOUNDS __launch_bounds__(S2Geo<N>::NT, CM_S2_MINB)
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

template <int N, int F>
__global__ void CM_S2_BOUNDS
stencil2_kernel(StencilParams<float> p, const __grid_constant__ CUtensorMap tmx,
                const __grid_constant__ CUtensorMap tmp, const __grid_constant__ CUtensorMap tmg,
                const __grid_constant__ CUtensorMap tma) {
    using G = S2Geo<N>;
    constexpr bool AUDIT = F & S2_AUDIT, PREV = AUDIT && (F & S2_PREV);
    constexpr bool TRACE = AUDIT && (F & S2_TRACE), STEP = F & S2_STEP, FISTA = F & S2_FISTA;
    constexpr unsigned USED = s2_used(F);
    constexpr int CI = G::CI, TJ = G::TJ, KC = G::KC, XW = G::XW, SW = G::SW;
    pdl_trigger();
    pdl_wait();
    if (p.st && ld_done(p.st)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* Sring = reinterpret_cast<float*>(smem_raw + G::OFF_S);   // [3][TJ+1][SW]
    double* red = reinterpret_cast<double*>(smem_raw + G::OFF_RED);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);
    const uint32_t smem_s = smem_u32(smem_raw), bar_s = smem_s + (uint32_t)G::OFF_BAR;

    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;  // w = row within tile, TJ = halo
    const bool halo = (w == TJ);
    // fp32 parameters as references into the (constant-bank) kernel parameters
    const float &eps = p.f_eps, &epsp = p.f_epsp, &mu = p.f_mu, &lr = p.f_lr, &lra = p.f_lra;
    const float &beta = p.f_beta, &g2 = p.f_g2, &inv2mu = p.f_inv2mu, &hmu = p.f_hmu;
    const float &cg = p.f_cg, &ce = p.f_ce;
    const bool has_beta = p.beta > 0.0, has_alpha = p.alpha > 0.0;
    constexpr bool with_prev = PREV;
    const bool convex = p.convex != 0;
    // s = 1/((g cg + ce) max(mu, g)): (cg, ce) = (1, eps') reweighted, (0, 1) convex
    const float theta = (FISTA && p.st) ? float(p.theta[p.st->iter - p.st->mom_base]) : 0.f;

    if (tid == 0) {
        for (int q = 0; q < G::NSTAGE; ++q) mbar_init(&bar[q], 1);
        mbar_fence_init();
    }
    // per-warp fp64 partial sums of the CTA's tiles (no fp64 registers held)
    for (int q = tid; q < 32 * NP1; q += blockDim.x) red[q] = 0.0;
    __syncthreads();

    // fp32 partials: fa over 8 planes, fb over the tile, then fp64 per warp
    float fa[NP1], fb[NP1];
#pragma unroll
    for (int q = 0; q < NP1; ++q) fa[q] = fb[q] = 0.f;

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
            tma_load_3d_s(ss, &tmx, i0 - 4, j0 - 1, q + zs, bs);
            if (with_prev) tma_load_3d_s(ss + (uint32_t)G::OFF_P, &tmp, i0 - 4, j0 - 1, q + zs, bs);
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
        }
        wait(k0 - 1);
        wait(k0);

        const int gj = j0 + w;                 // this warp's row (halo warp: j0 + TJ)
        const int ii = 4 * lane;
        const int gi0 = i0 + ii;
        const bool row_in = gj < N;
        // partial last x tile (N % 128 != 0): the lane's 4 voxels are all in or
        // all out; out-of-grid lanes keep s = 0 and join the shuffles, but load,
        // store and accumulate nothing
        const bool col_in = gi0 < N;
        // replicate boundary (gradient.cpp:7-24): the backward neighbour of the
        // first row / column / plane is the voxel itself, so D = 0 there without
        // a per-voxel test; forward terms vanish because s = 0 outside the grid
        const int ry = gj > 0 ? w : w + 1;     // slab row of j-1
        const bool xlo = (i0 == 0);
        // x slab row r (global j0 - 1 + r) of plane q, at this lane's 4 voxels
        auto xrow = [&](int q, int r) -> const float* {
            return reinterpret_cast<const float*>(stage(q)) + r * XW + 4 + ii;
        };
        // s on row w of plane q from the slabs of q and q-1 (rows w+1, w in slab coords)
        // returns s[4], plus |Dx|, d-sum for the voxels; halo column (i0+CI) via lane 31
        auto s_row = [&](int q, float (&xq)[4], float (&sv)[4], float (&gn)[4], float (&ds)[4]) {
            const float* xr = xrow(q, w + 1);
            const float* yr = xrow(q, ry);
            const float* zr = koff + q > 0 ? xrow(q - 1, w + 1) : xr;
            const float4 c4 = ld4(xr), y4 = ld4(yr), z4 = ld4(zr);
            xq[0] = c4.x; xq[1] = c4.y; xq[2] = c4.z; xq[3] = c4.w;
            const float yv[4] = {y4.x, y4.y, y4.z, y4.w}, zv[4] = {z4.x, z4.y, z4.z, z4.w};
            float xl = __shfl_up_sync(0xffffffffu, c4.w, 1);
            if (lane == 0) xl = xlo ? c4.x : xr[-1];
            const float xlv[4] = {xl, c4.x, c4.y, c4.z};
            const bool qin = koff + q < N && row_in && col_in;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float d1 = xq[c] - xlv[c], d2 = xq[c] - yv[c], d3 = xq[c] - zv[c];
                const float g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                const float mx = mu > g ? mu : g;
                const float s = rcp_(fmaf(g, cg, ce) * mx);  // convex: 1/mx
                sv[c] = qin ? s : 0.f;
                gn[c] = g;
                ds[c] = d1 + d2 + d3;
            }
        };
        // s on the column x = i0 + CI of tile row `lane` (0 .. TJ): computed by the
        // halo-row warp, so the row warps carry no divergent halo-column work
        auto s_col = [&](int q) -> float {
            const int r = lane, gjr = j0 + lane;
            if (r > TJ || koff + q >= N || gjr >= N || i0 + CI >= N) return 0.f;
            const float* xb = reinterpret_cast<const float*>(stage(q)) + 4 + CI;
            const float* zb = koff + q > 0 ? reinterpret_cast<const float*>(stage(q - 1)) + 4 + CI : xb;
            const float xc = xb[(r + 1) * XW];
            const float d1 = xc - xb[(r + 1) * XW - 1];
            const float d2 = xc - xb[(gjr > 0 ? r : r + 1) * XW];
            const float d3 = xc - zb[(r + 1) * XW];
            const float g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
            const float mx = fmaxf(mu, g);
            if (p.wtvf && !convex)
                return __ldg(p.wtvf + ((size_t)(q + zs) * N + gjr) * N + i0 + CI) * rcp_(mx);
            return rcp_(fmaf(g, cg, ce) * mx);
        };
        // per_m_step weights come from a frozen field: s uses w_tv from it
        auto apply_wtvf = [&](int q, float (&sv)[4], float (&gn)[4]) {
            if (!p.wtvf || convex || !(koff + q < N && row_in && col_in)) return;
            const float4 wv = __ldg(reinterpret_cast<const float4*>(
                p.wtvf + ((size_t)(q + zs) * N + gj) * N + gi0));
            const float wt[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float mx = mu > gn[c] ? mu : gn[c];
                sv[c] = wt[c] * rcp_(mx);
            }
        };

        // ---- prologue: s(., k0), rolling state of plane k0 and x_prev(k0-1)
        float x_cur[4], s_cur[4], gn_cur[4], ds_cur[4];
        s_row(k0, x_cur, s_cur, gn_cur, ds_cur);
        apply_wtvf(k0, s_cur, gn_cur);
        // s ring: plane k in slot (k - k0) % 3, rotated by pointer
        float* Sc_ring = Sring;                        // slot of plane k
        float* Sn_ring = Sring + G::SROW3;             // slot of plane k + 1
        float* Sx_ring = Sring + 2 * G::SROW3;         // the third slot
        float* S0 = Sc_ring;
        if (has_beta) {
            *reinterpret_cast<float4*>(S0 + w * SW + ii) =
                make_float4(s_cur[0], s_cur[1], s_cur[2], s_cur[3]);
            if (halo && lane <= TJ) S0[lane * SW + CI] = s_col(k0);
        }
        float xp_prev[4] = {0.f, 0.f, 0.f, 0.f};
        if (with_prev && !halo) {
            // plane k0-1 of x_prev (the plane itself at the global first plane)
            const float4 v = ld4(reinterpret_cast<const float*>(stage(koff + k0 > 0 ? k0 - 1 : k0) +
                                                                G::OFF_P) + (w + 1) * XW + 4 + ii);
            xp_prev[0] = v.x; xp_prev[1] = v.y; xp_prev[2] = v.z; xp_prev[3] = v.w;
        }
        __syncthreads();

        // one plane of the march; the rolling state alternates between two
        // register sets (the loop is unrolled by two) instead of being copied
        float x_nb[4], s_nb[4], gn_nb[4], ds_nb[4];
        auto step = [&](int k, float (&x_cur)[4], float (&s_cur)[4], float (&gn_cur)[4],
                        float (&ds_cur)[4], float (&x_nx)[4], float (&s_nx)[4],
                        float (&gn_nx)[4], float (&ds_nx)[4]) {
            if (tid == 0) issue(k + 2);  // slot of plane k-2: released by the previous barrier
            wait(k + 1);
            // ---- s of plane k+1 on this warp's row
            s_row(k + 1, x_nx, s_nx, gn_nx, ds_nx);
            apply_wtvf(k + 1, s_nx, gn_nx);
            float* Sn = Sn_ring;
            if (has_beta) {
                *reinterpret_cast<float4*>(Sn + w * SW + ii) =
                    make_float4(s_nx[0], s_nx[1], s_nx[2], s_nx[3]);
                if (halo && lane <= TJ) Sn[lane * SW + CI] = s_col(k + 1);
            }
            __syncthreads();
            if (!halo && row_in) {
                // ---- voxel (j, k): update, prox, partials
                const float* Sc = Sc_ring;
                const size_t gidx = ((size_t)(k + zs) * N + gj) * N + gi0;
                const unsigned char* stk = stage(k);
                const float4 g4 = ld4(reinterpret_cast<const float*>(stk + G::OFF_G) + w * CI + ii);
                const float4 a4 = ld4(reinterpret_cast<const float*>(stk + G::OFF_A) + w * CI + ii);
                const float gg[4] = {g4.x, g4.y, g4.z, g4.w}, av[4] = {a4.x, a4.y, a4.z, a4.w};
                float tvg[4] = {0.f, 0.f, 0.f, 0.f};
                if (has_beta) {
                    // x(j+1, k) and s(j+1, k): next row; x(i+1), s(i+1): next voxel
                    const float4 yp4 = ld4(xrow(k, w + 2));
                    const float4 sy4 = ld4(Sc + (w + 1) * SW + ii);
                    float xr4 = __shfl_down_sync(0xffffffffu, x_cur[0], 1);
                    float sr4 = __shfl_down_sync(0xffffffffu, s_cur[0], 1);
                    if (lane == 31) {
                        xr4 = xrow(k, w + 1)[4];          // x at i0 + CI
                        sr4 = Sc[w * SW + CI];
                    }
                    const float xn[4] = {x_cur[1], x_cur[2], x_cur[3], xr4};
                    const float sxv[4] = {s_cur[1], s_cur[2], s_cur[3], sr4};
                    const float yp[4] = {yp4.x, yp4.y, yp4.z, yp4.w};
                    const float sy[4] = {sy4.x, sy4.y, sy4.z, sy4.w};
#pragma unroll
                    for (int c = 0; c < 4; ++c)
                        tvg[c] = s_cur[c] * ds_cur[c] - sxv[c] * (xn[c] - x_cur[c]) -
                                 sy[c] * (yp[c] - x_cur[c]) - s_nx[c] * (x_nx[c] - x_cur[c]);
                }
                float wl1[4] = {1.f, 1.f, 1.f, 1.f}, wtv[4] = {1.f, 1.f, 1.f, 1.f};
                if (!convex) {
                    float ws[4] = {x_cur[0], x_cur[1], x_cur[2], x_cur[3]};
                    if (p.wl1src) {
                        if (p.wl1src == p.anchor) {
#pragma unroll
                            for (int c = 0; c < 4; ++c) ws[c] = av[c];
                        } else if (col_in) {
                            const float4 v = __ldg(reinterpret_cast<const float4*>(p.wl1src + gidx));
                            ws[0] = v.x; ws[1] = v.y; ws[2] = v.z; ws[3] = v.w;
                        }
                    }
                    if (p.wtvf) {
                        const float4 v = col_in ? __ldg(reinterpret_cast<const float4*>(p.wtvf + gidx))
                                                : make_float4(1.f, 1.f, 1.f, 1.f);
                        wtv[0] = v.x; wtv[1] = v.y; wtv[2] = v.z; wtv[3] = v.w;
#pragma unroll
                        for (int c = 0; c < 4; ++c) wl1[c] = rcp_(fabsf(ws[c]) + eps);
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float a = fabsf(ws[c]) + eps, b = gn_cur[c] + epsp;
                            const float r = rcp_(a * b);
                            wl1[c] = b * r;
                            wtv[c] = a * r;
                        }
                    }
                }
                float base[4] = {x_cur[0], x_cur[1], x_cur[2], x_cur[3]};
                if (FISTA && col_in) {
                    const float4 o4 = __ldg(reinterpret_cast<const float4*>(p.xold + gidx));
                    base[0] = o4.x; base[1] = o4.y; base[2] = o4.z; base[3] = o4.w;
                }
                float nx[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    float gs = 2.f * gg[c] + g2 * (x_cur[c] - av[c]);
                    if (has_beta) gs += beta * tvg[c];
                    float v = x_cur[c] - lr * gs;
                    if (has_alpha) {
                        const float th = lra * wl1[c];
                        // soft threshold, |v| <= th -> 0 (regularizer.cpp:107): v - clamp(v)
                        v = v - fminf(fmaxf(v, -th), th);
                    }
                    nx[c] = v;
                }
                if (!p.obj_only && col_in)
                    *reinterpret_cast<float4*>(p.xnext + gidx) = make_float4(nx[0], nx[1], nx[2], nx[3]);
                if (FISTA && !p.obj_only && col_in) {
                    float y[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) y[c] = nx[c] + theta * (nx[c] - base[c]);
                    *reinterpret_cast<float4*>(p.ynext + gidx) = make_float4(y[0], y[1], y[2], y[3]);
                }
                if (FISTA && col_in) {
                    // restart test (O'Donoghue & Candes): (y_k - x_{k+1}) . (x_{k+1} - x_k)
#pragma unroll
                    for (int c = 0; c < 4; ++c) fa[11] += (x_cur[c] - nx[c]) * (nx[c] - base[c]);
                }
                if (STEP && col_in) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float dx = nx[c] - base[c];
                        fa[9] += dx * dx;
                        fa[10] += nx[c] * nx[c];
                    }
                }
                if (AUDIT) {
                    float pl1[4] = {0.f, 0.f, 0.f, 0.f}, ptv[4] = {0.f, 0.f, 0.f, 0.f};
                    if (with_prev) {
                        const float* P = reinterpret_cast<const float*>(stk + G::OFF_P);
                        const float4 pc4 = ld4(P + (w + 1) * XW + 4 + ii);
                        const float4 py4 = ld4(P + ry * XW + 4 + ii);
                        float pm = __shfl_up_sync(0xffffffffu, pc4.w, 1);
                        if (lane == 0) pm = xlo ? pc4.x : P[(w + 1) * XW + 3];
                        const float pc[4] = {pc4.x, pc4.y, pc4.z, pc4.w};
                        const float pl[4] = {pm, pc4.x, pc4.y, pc4.z};
                        const float py[4] = {py4.x, py4.y, py4.z, py4.w};
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float e1 = pc[c] - pl[c], e2 = pc[c] - py[c], e3 = pc[c] - xp_prev[c];
                            const float a = fabsf(pc[c]) + eps;
                            const float b = sqrt_(e1 * e1 + e2 * e2 + e3 * e3) + epsp;
                            const float r = rcp_(a * b);
                            pl1[c] = b * r;
                            ptv[c] = a * r;
                            xp_prev[c] = pc[c];
                        }
                    }
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        if (!col_in) break;
                        const float ax = fabsf(x_cur[c]), g = gn_cur[c];
                        const float hb = g < mu ? g * g * inv2mu : g - hmu;
                        fa[0] += wl1[c] * ax;
                        fa[1] += wtv[c] * hb;
                        const float dd = x_cur[c] - av[c];
                        fa[5] += dd * dd;
                        if (with_prev) {
                            fa[6] += pl1[c] * ax;
                            fa[7] += ptv[c] * hb;
                        }
                        if (TRACE) {
                            fa[2] += wtv[c] * g;
                            fa[3] += __logf(ax + eps);
                            fa[4] += __logf(g + epsp);
                            if (with_prev) fa[8] += ptv[c] * g;
                        }
                    }
                }
            }
            float* const sfree = Sc_ring;
            Sc_ring = Sn_ring;
            Sn_ring = Sx_ring;
            Sx_ring = sfree;
        };
        for (int k = k0; k < k0 + KC; k += 2) {
            step(k, x_cur, s_cur, gn_cur, ds_cur, x_nb, s_nb, gn_nb, ds_nb);
            step(k + 1, x_nb, s_nb, gn_nb, ds_nb, x_cur, s_cur, gn_cur, ds_cur);
            if (USED && ((k + 1 - k0) & 7) == 7) {
#pragma unroll
                for (int q = 0; q < NP1; ++q)
                    if (USED & (1u << q)) {
                        fb[q] += fa[q];
                        fa[q] = 0.f;
                    }
            }
        }
        // tile partials -> this warp's fp64 slots (lane order fixed: deterministic)
        if constexpr (USED != 0) {
#pragma unroll
            for (int q = 0; q < NP1; ++q)
                if (USED & (1u << q)) {
                    const double v = warp_sum((double)fb[q]);
                    if (lane == 0) red[w * NP1 + q] += v;
                    fb[q] = 0.f;
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
inline int s2_flags(const StencilParams<float>& p) {
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

template <int N> inline cudaError_t stencil2_prepare() {
    cudaError_t e = cudaSuccess;
#define CM_S2_ATTR(FL)                                                                         \
    if (e == cudaSuccess)                                                                     \
        e = cudaFuncSetAttribute(stencil2_kernel<N, FL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)S2Geo<N>::SMEM);
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

template <int N>
inline cudaError_t stencil2_launch(StencilParams<float> p, int grid, cudaStream_t s,
                                   const CUtensorMap& tmx, const CUtensorMap& tmp,
                                   const CUtensorMap& tmg, const CUtensorMap& tma, bool pdl = false) {
    p.f_eps = float(p.eps);
    p.f_epsp = float(p.eps_prime);
    p.f_mu = float(p.mu);
    p.f_lr = float(p.lr);
    p.f_lra = float(p.lr * p.alpha);
    p.f_beta = float(p.beta);
    p.f_g2 = float(2.0 * p.gamma);
    p.f_inv2mu = float(0.5 / p.mu);
    p.f_hmu = float(0.5 * p.mu);
    p.f_cg = p.convex ? 0.f : 1.f;
    p.f_ce = p.convex ? 1.f : float(p.eps_prime);
    switch (s2_flags(p)) {
#define CM_S2_CASE(FL)                                                                         \
    case FL:                                                                                   \
        return launch_pdl(pdl, stencil2_kernel<N, FL>, dim3(grid), dim3(S2Geo<N>::NT),          \
                          S2Geo<N>::SMEM, s, p, tmx, tmp, tmg, tma);
        CM_S2_MODES(CM_S2_CASE)
#undef CM_S2_CASE
        default:
            return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int N> inline cudaError_t stencil2_occupancy(int* occ) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, stencil2_kernel<N, S2_AUDIT | S2_PREV>,
                                                         S2Geo<N>::NT, S2Geo<N>::SMEM);
}

} // namespace cm
