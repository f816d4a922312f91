// K1 fused (fp32, N in {256, 512}, one GPU): x-line C2R + stencil sweep +
// x-line R2C in ONE kernel, SURVEY §8(d)'s canonical K1.
//
// Reference loop replaced: regularizer.cpp:177-218 (one ISTA iteration's
// real-space part) with the inverse / forward x transforms of data_gradient
// (regularizer.cpp:87-101, fourier.cpp:18-31). The separate schedule wrote the
// data gradient g (4L bytes), read it back in the sweep (4L) and re-read
// x_{i+1} for the R2C (4L): 12L = 1.61 GB per 512^3 iteration. Here g and
// x_{i+1} never leave the chip:
//
//   * a thread-block CLUSTER of NCL = N/128 CTAs covers full x lines: CTA c
//     owns the x chunk [128c, 128c+128) of a TJ-row by KC-plane tile (the
//     stencil2 geometry: 4 row warps + 1 halo-row warp, x / x_{i-1} slabs and
//     anchor rows by TMA into a 4-deep ring) and the FFTs of TJ/NCL whole
//     lines (rows c*LPC .. c*LPC+LPC-1) per plane;
//   * C2R warp: the spectrum rows of its lines arrive by cp.async.bulk (4
//     planes ahead), are transformed in registers (split + half-length complex
//     FFT, xfft.cuh's math), scaled by 1/L and scattered as 128-float chunks to
//     the G ring of every CTA of the cluster with st.async (distributed shared
//     memory, mbarrier complete_tx on the receiver);
//   * stencil warps consume g from the G ring, write x_{i+1} (FISTA: also
//     y_{i+1}) to HBM once, and st.async their chunk of the new iterate (FISTA:
//     of y_{i+1}) into the line buffer of the CTA that owns the row's R2C;
//   * R2C warp: transforms the assembled lines and writes the packed spectrum
//     rows (in place: the C2R read of a row precedes its R2C write in the
//     same CTA through the barrier chain).
//   Flow control is by mbarriers only: g_full / ln_full (tx bytes from remote
//   st.async), g_empty / ln_empty (remote release arrivals, cluster scope).
//   The stencil warps synchronise among themselves with a named barrier; the
//   FFT warps never join it.
// HBM bytes per iteration of this kernel: spectrum 8H in and 8H out, x_i 4L,
// anchor 4L (+ x_{i-1} 4L in audit mode) in, x_{i+1} 4L out.
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "stencil2.cuh"
#include "tma.cuh"
#include "xfft.cuh"

namespace cm {

#ifndef CM_K1F_KC
#define CM_K1F_KC 32
#endif
#ifndef CM_K1F_NFFT
#define CM_K1F_NFFT 2  // warps per transform direction (planes alternate between them)
#endif
#ifndef CM_K1F_MINB
#define CM_K1F_MINB 2
#endif

template <int N> struct K1Geo {
    static constexpr bool OK = (N == 256 || N == 512);
    static constexpr int CI = 128, TJ = 4, KC = CM_K1F_KC;
    static constexpr int NCL = N / CI;             // CTAs per cluster (full x lines)
    static constexpr int LPC = TJ / NCL;           // FFT lines per CTA per plane
    static constexpr int NWS = TJ + 1;             // stencil warps (+ halo row)
    static constexpr int NF = CM_K1F_NFFT;         // C2R warps, then NF R2C warps
    static constexpr int WC2R = NWS, WR2C = NWS + NF;
    static constexpr int NT = (NWS + 2 * NF) * 32;
    static constexpr int NST = NWS * 32;           // threads of the stencil named barrier
    static constexpr int Nh = N / 2;
    static constexpr int E = Nh / 32;              // line elements per lane (one warp per line)
    static constexpr int XW = 136, XR = TJ + 2, PR = TJ + 1;
    static constexpr uint32_t XB = XR * XW * 4, PB = PR * XW * 4, AB = TJ * CI * 4;
    static constexpr size_t al(size_t v) { return (v + 127) / 128 * 128; }
    // x-slab stage ring (TMA; planes incl. the two ghost planes of a march)
    static constexpr size_t OFF_P = al(XB), OFF_A = al(OFF_P + PB);
    static constexpr size_t STAGE = al(OFF_A + AB);
    static constexpr int NSTAGE = 4;
    // G ring: g rows of this CTA's chunk, NG planes
    static constexpr int NG = 4;
    static constexpr size_t OFF_G = NSTAGE * STAGE;
    static constexpr size_t GSLOT = (size_t)TJ * CI * 4;
    // spectrum rows for the C2R warp, NL planes (LPC rows of Nh complex each)
    static constexpr int NL = 4;
    static constexpr size_t OFF_L = OFF_G + NG * GSLOT;
    static constexpr uint32_t LSLOT = (uint32_t)LPC * Nh * 8;
    // assembled real lines for the R2C warp, NLN planes (LPC lines of N floats)
    static constexpr int NLN = 4;
    static constexpr size_t OFF_LN = OFF_L + NL * (size_t)LSLOT;
    static constexpr uint32_t LNSLOT = (uint32_t)LPC * N * 4;
    // s ring, FFT exchange buffers, twiddles, reductions, barriers
    static constexpr int SW = CI + 4;
    static constexpr size_t SROW3 = (size_t)(TJ + 1) * SW;
    static constexpr size_t OFF_S = al(OFF_LN + NLN * (size_t)LNSLOT);
    static constexpr int PADX = (Nh + (Nh >> 3) + 2) / 2 * 2;
    static constexpr size_t OFF_X = al(OFF_S + 3 * SROW3 * 4);   // [2 NF warps][PADX] complex
    static constexpr size_t OFF_TW = OFF_X + 2 * NF * (size_t)PADX * 8;
    static constexpr size_t OFF_RED = al(OFF_TW + (size_t)N * 8);
    static constexpr size_t OFF_BAR = OFF_RED + 8 * NP1 * 8;
    // barriers: stage[4] g_full[4] g_empty[4] l_full[4] ln_full[NLN] ln_empty[NLN]
    static constexpr int B_STAGE = 0, B_GF = 4, B_GE = 8, B_LF = 12, B_LNF = 16, B_LNE = 16 + NLN,
                         NBAR = 16 + 2 * NLN;
    static constexpr size_t SMEM = OFF_BAR + NBAR * 8;
    static constexpr int NTJ = N / TJ, NTK = N / KC;
    static_assert(NL % NF == 0 && NLN % NF == 0 && NG % NF == 0, "rings are split by plane parity");
    static constexpr int NTILES = NTJ * NTK;       // cluster tiles (j block, k block)
};

// ---- cluster / distributed-shared-memory primitives (inline PTX, sm_90+) ----
__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa_s(uint32_t addr, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::
                     : "memory");
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(
            raddr),
        "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, float2 v, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];" ::"r"(
                     raddr),
                 "f"(v.x), "f"(v.y), "r"(rbar)
                 : "memory");
}
// relaxed arrival on a (possibly remote) barrier of the cluster. The arrivals
// only say "this slot's data has been consumed" (its shared-memory reads have
// returned and fed arithmetic before the arrive issues); a release here would
// be a cluster-scope fence that waits for the thread's outstanding HBM stores
// (ncu: `membar` stalls dominated the first version of this kernel).
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t rbar) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
#ifndef CM_K1F_SPIN_TRAP
#define CM_K1F_SPIN_TRAP (1u << 30)  // a wait this long is a bug: trap instead of hanging the GPU
#endif
// Waits on barriers completed from OTHER CTAs of the cluster (st.async tx,
// remote arrivals). A blocking try_wait may suspend the warp for up to a
// system-dependent time and is not promptly woken by remote completions, so
// these waits poll: test_wait (CM_K1F_WAIT 2, default) or try_wait with a
// short suspend-time hint (1) or the default try_wait (0).
#ifndef CM_K1F_WAIT
#define CM_K1F_WAIT 2
#endif
#ifndef CM_K1F_HINT
#define CM_K1F_HINT 32
#endif
__device__ __forceinline__ void mbar_wait_cl(uint32_t bar, uint32_t parity) {
    uint32_t ok = 0, spins = 0;
    do {
#if CM_K1F_WAIT == 2
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
#elif CM_K1F_WAIT == 1
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity), "r"(CM_K1F_HINT)
            : "memory");
#else
        asm volatile(
            "{\n.reg .pred P1;\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
            "selp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(bar), "r"(parity)
            : "memory");
#endif
        if (!ok && ++spins > CM_K1F_SPIN_TRAP) __trap();
    } while (!ok);
}
__device__ __forceinline__ void bulk_load_s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void named_bar(int id, int count) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

#ifdef CM_K1F_TRACE
__device__ unsigned long long* g_k1f_trace;
#define K1T(ev, uu)                                                                            \
    do {                                                                                       \
        if (lane == 0 && blockIdx.x < (unsigned)NCL && (uu) < 64) {                            \
            unsigned long long t_;                                                             \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
            g_k1f_trace[((size_t)blockIdx.x * 10 + (ev)) * 64 + (uu)] = t_;                    \
        }                                                                                      \
    } while (0)
#else
#define K1T(ev, uu) do {} while (0)
#endif

template <int N, int F>
__global__ void __launch_bounds__(K1Geo<N>::NT, CM_K1F_MINB)
k1f_kernel(StencilParams<float> p, float2* __restrict__ S, const float2* __restrict__ twN, float invL,
           const __grid_constant__ CUtensorMap tmx, const __grid_constant__ CUtensorMap tmp,
           const __grid_constant__ CUtensorMap tma) {
    using G = K1Geo<N>;
    using C = float2;
    constexpr bool AUDIT = F & S2_AUDIT, PREV = AUDIT && (F & S2_PREV);
    constexpr bool TRACE = AUDIT && (F & S2_TRACE), STEP = F & S2_STEP, FISTA = F & S2_FISTA;
    constexpr unsigned USED = s2_used(F);
    constexpr int CI = G::CI, TJ = G::TJ, KC = G::KC, XW = G::XW, SW = G::SW, NCL = G::NCL;
    constexpr int LPC = G::LPC, Nh = G::Nh, E = G::E;
    if (p.st && ld_done(p.st)) return;  // uniform over the cluster
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float* Sring = reinterpret_cast<float*>(smem_raw + G::OFF_S);
    double* red = reinterpret_cast<double*>(smem_raw + G::OFF_RED);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);
    const uint32_t smem_s = smem_u32(smem_raw), bar_s = smem_s + (uint32_t)G::OFF_BAR;
    auto B = [&](int i) { return bar_s + 8u * (uint32_t)i; };
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const uint32_t crank = cluster_rank();
    const int cid = blockIdx.x / NCL, ncls = gridDim.x / NCL;
    const int i0 = (int)crank * CI;
    C* tw = reinterpret_cast<C*>(smem_raw + G::OFF_TW);
    stage_table(tw, twN, N);
    if (tid == 0) {
        for (int q = 0; q < G::NSTAGE; ++q) mbar_init(&bar[G::B_STAGE + q], 1);
        for (int q = 0; q < G::NG; ++q) {
            mbar_init(&bar[G::B_GF + q], 1);    // armed by this CTA's thread 0 (expect_tx)
            mbar_init(&bar[G::B_GE + q], NCL);  // one release per consumer CTA
        }
        for (int q = 0; q < G::NL; ++q) mbar_init(&bar[G::B_LF + q], 1);
        for (int q = 0; q < G::NLN; ++q) {
            mbar_init(&bar[G::B_LNF + q], 1);   // armed by the R2C warp
            mbar_init(&bar[G::B_LNE + q], NCL); // one release per R2C owner CTA
        }
        mbar_fence_init();
        // arm the first phase of every G / line slot: NCL producers deliver TJ rows
        for (int q = 0; q < G::NG; ++q) mbar_expect_tx_s(B(G::B_GF + q), (uint32_t)G::GSLOT);
        for (int q = 0; q < G::NLN; ++q) mbar_expect_tx_s(B(G::B_LNF + q), G::LNSLOT);
    }
    for (int q = tid; q < 8 * NP1; q += blockDim.x) red[q] = 0.0;
    __syncthreads();
    cluster_sync_all();  // every CTA's barriers exist before any remote access

    const int ntiles_c = G::NTILES;
    // plane stream of this cluster: u = (tile ordinal) * KC + (k - k0)
    auto tile_of = [&](int ord) { return cid + ord * ncls; };
    auto tile_jk = [&](int tile, int& j0, int& k0) {
        j0 = (tile % G::NTJ) * TJ;
        k0 = (tile / G::NTJ) * KC;
    };

    if (w >= G::WC2R && w < G::WC2R + G::NF) {
        const int f = w - G::WC2R;  // this warp's planes: u = f (mod NF)
        // ============================ C2R warp ============================
        const uint32_t lbase = smem_s + (uint32_t)G::OFF_L;
        C* xb = reinterpret_cast<C*>(smem_raw + G::OFF_X) + f * G::PADX;
        const PadAddr pad{};
        const WarpSync wsync{};
        auto issue_line = [&](int u) {  // spectrum rows of plane u -> line slot u % NL
            const int ord = u / KC, tile = tile_of(ord);
            if (tile >= ntiles_c) return;
            int j0, k0;
            tile_jk(tile, j0, k0);
            const int k = k0 + u % KC;
            const int sl = u % G::NL;
            mbar_expect_tx_s(B(G::B_LF + sl), G::LSLOT);
            const C* src = S + ((size_t)k * N + j0 + (int)crank * LPC) * Nh;  // LPC rows, contiguous
            bulk_load_s(lbase + (uint32_t)sl * G::LSLOT, src, G::LSLOT, B(G::B_LF + sl));
        };
        if (lane == 0)
            for (int u = f; u < G::NL; u += G::NF) issue_line(u);
        for (int u = f;; u += G::NF) {
            const int ord = u / KC, tile = tile_of(ord);
            if (tile >= ntiles_c) break;
            const int sl = u % G::NL;
            mbar_wait_cl(B(G::B_LF + sl), (uint32_t)(u / G::NL) & 1u);
            K1T(4, u);
            const C* lsrc = reinterpret_cast<const C*>(smem_raw + G::OFF_L + (size_t)sl * G::LSLOT);
            C v[LPC][E];
#pragma unroll
            for (int l = 0; l < LPC; ++l)
#pragma unroll
                for (int m = 0; m < E; ++m) v[l][m] = lsrc[l * Nh + lane + 32 * m];
            __syncwarp();
            if (lane == 0) issue_line(u + G::NL);  // the slot's data is in registers
            const int gs = u % G::NG;
#pragma unroll
            for (int l = 0; l < LPC; ++l) {
                // split the packed half spectrum into the N/2-point complex
                // sequence of the real line (xfft.cuh DIR 0)
#pragma unroll
                for (int m = 0; m < E; ++m) xb[pad(lane + 32 * m)] = v[l][m];
                __syncwarp();
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = lane + 32 * m;
                    const C q = v[l][m];
                    if (hh == 0) {
                        v[l][m] = make_float2(q.x + q.y, q.x - q.y);
                    } else {
                        const C qm = xb[pad(Nh - hh)];
                        const C a = make_float2(q.x + qm.x, q.y - qm.y);
                        const C d = make_float2(q.x - qm.x, q.y + qm.y);
                        const C bb = cmulc(d, tw[hh]);
                        v[l][m] = make_float2(a.x - bb.y, a.y + bb.x);
                    }
                }
                __syncwarp();
                fft_regs<Nh, E, N, false>(v[l], lane, xb, pad, xline_tw<float, false>(tw, nullptr),
                                          wsync);
                __syncwarp();
            }
            // g chunks to every CTA of the cluster once its G slot is free
            K1T(5, u);
            mbar_wait_cl(B(G::B_GE + gs), ((uint32_t)(u / G::NG) & 1u) ^ 1u);
            K1T(6, u);
#pragma unroll
            for (int l = 0; l < LPC; ++l) {
                const int row = (int)crank * LPC + l;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    // x = 2(lane + 32 m): chunk c = m / 2, local x = 2 lane + 64 (m % 2)
                    const uint32_t c = (uint32_t)(m / 2);
                    const uint32_t off = (uint32_t)(G::OFF_G + gs * G::GSLOT) +
                                         4u * (uint32_t)(row * CI + 2 * lane + 64 * (m % 2));
                    st_async_v2(mapa_s(smem_s + off, c),
                                make_float2(v[l][m].x * invL, v[l][m].y * invL),
                                mapa_s(B(G::B_GF + gs), c));
                }
            }
        }
    } else if (w >= G::WR2C) {
        const int f = w - G::WR2C;
        // ============================ R2C warp ============================
        C* xb = reinterpret_cast<C*>(smem_raw + G::OFF_X) + (G::NF + f) * G::PADX;
        const PadAddr pad{};
        const WarpSync wsync{};
        for (int u = f;; u += G::NF) {
            const int ord = u / KC, tile = tile_of(ord);
            if (tile >= ntiles_c) break;
            int j0, k0;
            tile_jk(tile, j0, k0);
            const int k = k0 + u % KC;
            const int sl = u % G::NLN;
            mbar_wait_cl(B(G::B_LNF + sl), (uint32_t)(u / G::NLN) & 1u);
            K1T(7, u);
            const float* lsrc = reinterpret_cast<const float*>(smem_raw + G::OFF_LN + (size_t)sl * G::LNSLOT);
            C v[LPC][E];
#pragma unroll
            for (int l = 0; l < LPC; ++l)
#pragma unroll
                for (int m = 0; m < E; ++m)
                    v[l][m] = *reinterpret_cast<const C*>(lsrc + l * N + 2 * (lane + 32 * m));
            __syncwarp();
#pragma unroll
            for (int l = 0; l < LPC; ++l) {
                fft_regs<Nh, E, N, true>(v[l], lane, xb, pad, xline_tw<float, true>(tw, nullptr), wsync);
                __syncwarp();
                if (l == LPC - 1 && lane == 0) {
                    // every read of the slot has fed the transforms: re-arm it for
                    // plane u + NLN, then release it to every writer
                    mbar_expect_tx_s(B(G::B_LNF + sl), G::LNSLOT);
                    for (int c = 0; c < NCL; ++c) mbar_arrive_cluster(mapa_s(B(G::B_LNE + sl), (uint32_t)c));
                }
#pragma unroll
                for (int m = 0; m < E; ++m) xb[pad(lane + 32 * m)] = v[l][m];
                __syncwarp();
                C* Srow = S + ((size_t)k * N + j0 + (int)crank * LPC + l) * Nh;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = lane + 32 * m;
                    const C z = v[l][m];
                    C out;
                    if (hh == 0) {
                        out = make_float2(z.x + z.y, z.x - z.y);  // X(0) + i X(N/2)
                    } else {
                        const C zm = xb[pad(Nh - hh)];
                        const C e = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
                        const C o = make_float2(0.5f * (z.y + zm.y), -0.5f * (z.x - zm.x));
                        out = cadd(e, cmul(o, tw[hh]));
                    }
                    Srow[hh] = out;
                }
                __syncwarp();
            }
            K1T(8, u);
        }
    } else {
        // ========================= stencil warps =========================
        const bool halo = (w == TJ);
        const float &eps = p.f_eps, &epsp = p.f_epsp, &mu = p.f_mu, &lr = p.f_lr, &lra = p.f_lra;
        const float &beta = p.f_beta, &g2 = p.f_g2, &inv2mu = p.f_inv2mu, &hmu = p.f_hmu;
        const float &cg = p.f_cg, &ce = p.f_ce;
        const bool has_beta = p.beta > 0.0, has_alpha = p.alpha > 0.0;
        constexpr bool with_prev = PREV;
        const bool convex = p.convex != 0;
        const float theta = (FISTA && p.st) ? float(p.theta[p.st->iter - p.st->mom_base]) : 0.f;
        float fa[NP1], fb[NP1];
#pragma unroll
        for (int q = 0; q < NP1; ++q) fa[q] = fb[q] = 0.f;
        uint32_t phase_bits = 0;
        const float* Gring = reinterpret_cast<const float*>(smem_raw + G::OFF_G);
        int u = 0;  // march-plane counter (the cluster's plane stream)
        for (int ord = 0;; ++ord) {
            const int tile = tile_of(ord);
            if (tile >= ntiles_c) break;
            int j0, k0;
            tile_jk(tile, j0, k0);
            auto slot_of = [&](int q) { return (q - k0 + 1) & (G::NSTAGE - 1); };
            auto stage = [&](int q) { return smem_raw + (size_t)slot_of(q) * G::STAGE; };
            auto issue = [&](int q) {
                if (q > k0 + KC) return;
                const int sl = slot_of(q);
                const uint32_t bs = B(G::B_STAGE + sl), ss = smem_s + (uint32_t)((size_t)sl * G::STAGE);
                mbar_expect_tx_s(bs, G::XB + (with_prev ? G::PB : 0u) + G::AB);
                tma_load_3d_s(ss, &tmx, i0 - 4, j0 - 1, q, bs);
                if (with_prev) tma_load_3d_s(ss + (uint32_t)G::OFF_P, &tmp, i0 - 4, j0 - 1, q, bs);
                tma_load_3d_s(ss + (uint32_t)G::OFF_A, &tma, i0, j0, q, bs);
            };
            auto wait = [&](int q) {
                const int sl = slot_of(q);
                mbar_wait_s(B(G::B_STAGE + sl), (phase_bits >> sl) & 1u);
                phase_bits ^= (1u << sl);
            };
            // release the G slot of march plane uu to every C2R producer; arm its next phase
            auto release_g = [&](int uu) {
                const int gs = uu % G::NG;
                mbar_expect_tx_s(B(G::B_GF + gs), (uint32_t)G::GSLOT);
                for (int c = 0; c < NCL; ++c) mbar_arrive_cluster(mapa_s(B(G::B_GE + gs), (uint32_t)c));
            };
            if (tid == 0) {
                issue(k0 - 1);
                issue(k0);
                issue(k0 + 1);
            }
            wait(k0 - 1);
            wait(k0);

            const int gj = j0 + w;
            const int ii = 4 * lane;
            const int gi0 = i0 + ii;
            const bool row_in = gj < N;
            const int ry = gj > 0 ? w : w + 1;
            const bool xlo = (i0 == 0);
            auto xrow = [&](int q, int r) -> const float* {
                return reinterpret_cast<const float*>(stage(q)) + r * XW + 4 + ii;
            };
            auto s_row = [&](int q, float (&xq)[4], float (&sv)[4], float (&gn)[4], float (&ds)[4]) {
                const float* xr = xrow(q, w + 1);
                const float* yr = xrow(q, ry);
                const float* zr = q > 0 ? xrow(q - 1, w + 1) : xr;
                const float4 c4 = ld4(xr), y4 = ld4(yr), z4 = ld4(zr);
                xq[0] = c4.x; xq[1] = c4.y; xq[2] = c4.z; xq[3] = c4.w;
                const float yv[4] = {y4.x, y4.y, y4.z, y4.w}, zv[4] = {z4.x, z4.y, z4.z, z4.w};
                float xl = __shfl_up_sync(0xffffffffu, c4.w, 1);
                if (lane == 0) xl = xlo ? c4.x : xr[-1];
                const float xlv[4] = {xl, c4.x, c4.y, c4.z};
                const bool qin = q < N && row_in;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float d1 = xq[c] - xlv[c], d2 = xq[c] - yv[c], d3 = xq[c] - zv[c];
                    const float g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                    const float mx = mu > g ? mu : g;
                    const float s = rcp_(fmaf(g, cg, ce) * mx);
                    sv[c] = qin ? s : 0.f;
                    gn[c] = g;
                    ds[c] = d1 + d2 + d3;
                }
            };
            auto s_col = [&](int q) -> float {
                const int r = lane, gjr = j0 + lane;
                if (r > TJ || q >= N || gjr >= N || i0 + CI >= N) return 0.f;
                const float* xb = reinterpret_cast<const float*>(stage(q)) + 4 + CI;
                const float* zb = q > 0 ? reinterpret_cast<const float*>(stage(q - 1)) + 4 + CI : xb;
                const float xc = xb[(r + 1) * XW];
                const float d1 = xc - xb[(r + 1) * XW - 1];
                const float d2 = xc - xb[(gjr > 0 ? r : r + 1) * XW];
                const float d3 = xc - zb[(r + 1) * XW];
                const float g = sqrt_(d1 * d1 + d2 * d2 + d3 * d3);
                const float mx = fmaxf(mu, g);
                if (p.wtvf && !convex)
                    return __ldg(p.wtvf + ((size_t)q * N + gjr) * N + i0 + CI) * rcp_(mx);
                return rcp_(fmaf(g, cg, ce) * mx);
            };
            auto apply_wtvf = [&](int q, float (&sv)[4], float (&gn)[4]) {
                if (!p.wtvf || convex || !(q < N && row_in)) return;
                const float4 wv = __ldg(reinterpret_cast<const float4*>(p.wtvf + ((size_t)q * N + gj) * N + gi0));
                const float wt[4] = {wv.x, wv.y, wv.z, wv.w};
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const float mx = mu > gn[c] ? mu : gn[c];
                    sv[c] = wt[c] * rcp_(mx);
                }
            };

            float x_cur[4], s_cur[4], gn_cur[4], ds_cur[4];
            s_row(k0, x_cur, s_cur, gn_cur, ds_cur);
            apply_wtvf(k0, s_cur, gn_cur);
            float* Sc_ring = Sring;
            float* Sn_ring = Sring + G::SROW3;
            float* Sx_ring = Sring + 2 * G::SROW3;
            if (has_beta) {
                *reinterpret_cast<float4*>(Sc_ring + w * SW + ii) = make_float4(s_cur[0], s_cur[1], s_cur[2], s_cur[3]);
                if (halo && lane <= TJ) Sc_ring[lane * SW + CI] = s_col(k0);
            }
            float xp_prev[4] = {0.f, 0.f, 0.f, 0.f};
            if (with_prev && !halo) {
                const float4 v = ld4(reinterpret_cast<const float*>(stage(k0 > 0 ? k0 - 1 : k0) + G::OFF_P) +
                                     (w + 1) * XW + 4 + ii);
                xp_prev[0] = v.x; xp_prev[1] = v.y; xp_prev[2] = v.z; xp_prev[3] = v.w;
            }
            named_bar(1, G::NST);

            float x_nb[4], s_nb[4], gn_nb[4], ds_nb[4];
            auto step = [&](int k, float (&x_cur)[4], float (&s_cur)[4], float (&gn_cur)[4],
                            float (&ds_cur)[4], float (&x_nx)[4], float (&s_nx)[4], float (&gn_nx)[4],
                            float (&ds_nx)[4]) {
                if (w == 0) K1T(0, u);
                if (tid == 0) issue(k + 2);
                wait(k + 1);
                s_row(k + 1, x_nx, s_nx, gn_nx, ds_nx);
                apply_wtvf(k + 1, s_nx, gn_nx);
                float* Sn = Sn_ring;
                if (has_beta) {
                    *reinterpret_cast<float4*>(Sn + w * SW + ii) = make_float4(s_nx[0], s_nx[1], s_nx[2], s_nx[3]);
                    if (halo && lane <= TJ) Sn[lane * SW + CI] = s_col(k + 1);
                }
                named_bar(1, G::NST);
                if (w == 0) K1T(1, u);
                // the previous plane's G slot is consumed by every stencil warp
                if (tid == 0 && k > k0) release_g(u - 1);
                if (!halo && row_in) {
                    const int gs = u % G::NG;
                    mbar_wait_cl(B(G::B_GF + gs), (uint32_t)(u / G::NG) & 1u);
                    if (w == 0) K1T(2, u);
                    const float* Sc = Sc_ring;
                    const size_t gidx = ((size_t)k * N + gj) * N + gi0;
                    const unsigned char* stk = stage(k);
                    const float4 g4 = ld4(Gring + (size_t)gs * TJ * CI + w * CI + ii);
                    const float4 a4 = ld4(reinterpret_cast<const float*>(stk + G::OFF_A) + w * CI + ii);
                    const float gg[4] = {g4.x, g4.y, g4.z, g4.w}, av[4] = {a4.x, a4.y, a4.z, a4.w};
                    float tvg[4] = {0.f, 0.f, 0.f, 0.f};
                    if (has_beta) {
                        const float4 yp4 = ld4(xrow(k, w + 2));
                        const float4 sy4 = ld4(Sc + (w + 1) * SW + ii);
                        float xr4 = __shfl_down_sync(0xffffffffu, x_cur[0], 1);
                        float sr4 = __shfl_down_sync(0xffffffffu, s_cur[0], 1);
                        if (lane == 31) {
                            xr4 = xrow(k, w + 1)[4];
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
                            } else {
                                const float4 v = __ldg(reinterpret_cast<const float4*>(p.wl1src + gidx));
                                ws[0] = v.x; ws[1] = v.y; ws[2] = v.z; ws[3] = v.w;
                            }
                        }
                        if (p.wtvf) {
                            const float4 v = __ldg(reinterpret_cast<const float4*>(p.wtvf + gidx));
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
                    if (FISTA) {
                        const float4 o4 = __ldg(reinterpret_cast<const float4*>(p.xold + gidx));
                        base[0] = o4.x; base[1] = o4.y; base[2] = o4.z; base[3] = o4.w;
                    }
                    float nx[4];
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float gsum = 2.f * gg[c] + g2 * (x_cur[c] - av[c]);
                        if (has_beta) gsum += beta * tvg[c];
                        float v = x_cur[c] - lr * gsum;
                        if (has_alpha) {
                            const float th = lra * wl1[c];
                            v = v - fminf(fmaxf(v, -th), th);
                        }
                        nx[c] = v;
                    }
                    *reinterpret_cast<float4*>(p.xnext + gidx) = make_float4(nx[0], nx[1], nx[2], nx[3]);
                    float4 spec = make_float4(nx[0], nx[1], nx[2], nx[3]);  // the next spectrum's source
                    if (FISTA) {
                        float y[4];
#pragma unroll
                        for (int c = 0; c < 4; ++c) y[c] = nx[c] + theta * (nx[c] - base[c]);
                        spec = make_float4(y[0], y[1], y[2], y[3]);
                        *reinterpret_cast<float4*>(p.ynext + gidx) = spec;
                    }
                    // this row's chunk of the new line -> the CTA that owns its R2C
                    {
                        const int ls = u % G::NLN;
                        mbar_wait_cl(B(G::B_LNE + ls), ((uint32_t)(u / G::NLN) & 1u) ^ 1u);
                        if (w == 0) K1T(3, u);
                        const uint32_t owner = (uint32_t)(w / LPC);
                        const uint32_t off = (uint32_t)(G::OFF_LN + ls * G::LNSLOT) +
                                             4u * (uint32_t)((w % LPC) * N + i0 + ii);
                        st_async_v4(mapa_s(smem_s + off, owner), spec, mapa_s(B(G::B_LNF + ls), owner));
                    }
                    if (STEP) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) {
                            const float dx = nx[c] - base[c];
                            fa[9] += dx * dx;
                            fa[10] += nx[c] * nx[c];
                        }
                    }
                    if (FISTA) {
#pragma unroll
                        for (int c = 0; c < 4; ++c) fa[11] += (x_cur[c] - nx[c]) * (nx[c] - base[c]);
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
                ++u;
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
            if constexpr (USED != 0) {
#pragma unroll
                for (int q = 0; q < NP1; ++q)
                    if (USED & (1u << q)) {
                        const double v = warp_sum((double)fb[q]);
                        if (lane == 0) red[w * NP1 + q] += v;
                        fb[q] = 0.f;
                    }
            }
            named_bar(1, G::NST);
            if (tid == 0) release_g(u - 1);  // the tile's last plane
        }
    }
    __syncthreads();
    if (p.part && tid < NP1) {
        double t = 0.0;
        for (int v = 0; v < G::NWS; ++v) t += red[v * NP1 + tid];
        p.part[(size_t)blockIdx.x * NP1 + tid] = t;
    }
    cluster_sync_all();  // no CTA leaves while a peer may still address its shared memory
}

template <int N> inline cudaError_t k1f_prepare() {
    cudaError_t e = cudaSuccess;
#define CM_K1F_ATTR(FL)                                                                          \
    if (e == cudaSuccess)                                                                       \
        e = cudaFuncSetAttribute(k1f_kernel<N, FL>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)K1Geo<N>::SMEM);                                          \
    if (e == cudaSuccess)                                                                       \
        e = cudaFuncSetAttribute(k1f_kernel<N, FL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    CM_S2_MODES(CM_K1F_ATTR)
#undef CM_K1F_ATTR
    return e;
}

template <int N> inline cudaLaunchConfig_t k1f_config(int grid, cudaStream_t s, cudaLaunchAttribute* at) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(K1Geo<N>::NT);
    cfg.dynamicSmemBytes = K1Geo<N>::SMEM;
    cfg.stream = s;
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = K1Geo<N>::NCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cfg;
}

// clusters that fit at once (persistent grid = that many clusters, capped by the tiles)
template <int N> inline int k1f_grid(cudaStream_t s) {
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = k1f_config<N>(K1Geo<N>::NCL, s, at);
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, k1f_kernel<N, S2_AUDIT | S2_PREV>, &cfg) != cudaSuccess ||
        ncl < 1) {
        cudaGetLastError();
        return 0;
    }
    return std::min(ncl, K1Geo<N>::NTILES) * K1Geo<N>::NCL;
}

template <int N>
inline cudaError_t k1f_launch(StencilParams<float> p, float2* S, const float2* twN, int grid,
                              cudaStream_t s, const CUtensorMap& tmx, const CUtensorMap& tmp,
                              const CUtensorMap& tma) {
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
    const float invL = float(1.0 / ((double)N * N * N));
    cudaLaunchAttribute at[1];
    cudaLaunchConfig_t cfg = k1f_config<N>(grid, s, at);
#ifdef CM_K1F_TRACE
    static unsigned long long* tbuf = nullptr;
    static int launches = 0;
    const size_t tn = (size_t)K1Geo<N>::NCL * 10 * 64;
    if (!tbuf) {
        cudaMalloc(&tbuf, tn * 8);
        cudaMemcpyToSymbol(g_k1f_trace, &tbuf, sizeof(tbuf));
    }
    cudaMemsetAsync(tbuf, 0, tn * 8, s);
#endif
    cudaError_t rc = cudaErrorInvalidValue;
    switch (s2_flags(p)) {
#define CM_K1F_CASE(FL) \
    case FL:            \
        rc = cudaLaunchKernelEx(&cfg, k1f_kernel<N, FL>, p, S, twN, invL, tmx, tmp, tma); \
        break;
        CM_S2_MODES(CM_K1F_CASE)
#undef CM_K1F_CASE
        default:
            break;
    }
#ifdef CM_K1F_TRACE
    if (++launches == 2) {
        std::vector<unsigned long long> h(tn);
        cudaMemcpyAsync(h.data(), tbuf, tn * 8, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        unsigned long long t0 = ~0ull;
        for (auto v : h) if (v && v < t0) t0 = v;
        for (int b = 0; b < K1Geo<N>::NCL; ++b)
            for (int ev = 0; ev < 9; ++ev) {
                std::fprintf(stderr, "cta%d ev%d:", b, ev);
                for (int u = 0; u < 40; ++u) {
                    const unsigned long long v = h[((size_t)b * 10 + ev) * 64 + u];
                    std::fprintf(stderr, " %lld", v ? (long long)(v - t0) : -1ll);
                }
                std::fprintf(stderr, "\n");
            }
    }
#endif
    return rc;
}

} // namespace cm
