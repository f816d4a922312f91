// K3 — z pass with the Fourier-diagonal data term fused (sm_100a).
//
// zmain_kernel: FFT along k of TWY consecutive half-spectrum columns h at one
//   row b (the y-pass tile shape: coalesced rows, registers in, registers out),
//   then per element G = W F - Yh (regularizer.cpp:91-92 with the phase sign
//   folded into Yh), the fit partials (regularizer.cpp:114-123,
//   weight 2 for 0 < h < N/2) and the inverse FFT along k.
// zcol0_kernel: the packed column h = 0 carries F(0,b,c) + i F(N/2,b,c); its two
//   Hermitian planes are separated with the Friedel mate (-b,-c), multiplied
//   and repacked. zmain leaves the forward-transformed column in Z0[b][c]; one
//   block per mate pair (b, -b) finishes it (1/Nh of the data).
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace cm {

template <typename R> struct ZMParams {
    using C = Cx<R>;
    C* S;
    C* Z0;          // [N][N] forward-transformed packed column 0 (b major)
    const R* W;
    const R* Wn;
    const C* Yh;
    const C* Yn;
    const C* twN;
    const float4* twF4; // packed forward / inverse tables (fp32)
    const float4* twI4;
    double* part;   // [nblocks_main + N/2 + 1][NP3]
    DevState* st;
    int nrows;      // rows b of the spectrum block (N, or NB on a b-slab rank)
    // column-0 inputs row-major for the column-0 kernels: Q0[(b*N + c)*3 + j] =
    // {(W(0), W(N/2)), Yh(0), Y(N/2)} (the h = 0 entries of W/Yh are strided)
    const Cx<R>* Q0;
    // b-slab ranks with split column halves: stored row length and the first
    // (global) column of this launch; one GPU: N/2 and 0 (compile-time there)
    int hlen, h0;
    // one GPU: L2 prefetch lookahead in tiles for S (rows of tile + pf) and for
    // the contiguous W / Yh tiles (tile + pfw; -1: off); 0 / -1 disable
    int pf = 0, pfw = -1;
    // one GPU, fp32: S as a 3D tensor map (float pairs) with z boxes {2 TW, 1, <= 256}
    // in global memory; the S prefetch of tile + pf is then one TMA
    // cp.async.bulk.prefetch.tensor per 256 rows instead of one LSU prefetch per row
    const CUtensorMap* tmS = nullptr;
};

#ifndef CM_Z_E8
#define CM_Z_E8 1
#endif
#ifndef CM_Z_E16
#define CM_Z_E16 1
#endif
#ifndef CM_Z_E16_MIN
#define CM_Z_E16_MIN 512
#endif
#ifndef CM_Z_E32_MIN
#define CM_Z_E32_MIN 1024  // 1024^3: z pass 5.5 -> 4.2 ms per iteration
#endif
#ifndef CM_Z_TW
#define CM_Z_TW 0  // columns per CTA (0: 16, capped at 1024 threads)
#endif
#ifndef CM_Z_WBULK
#define CM_Z_WBULK 0  // measured slower at 512^3 (0.49 vs 0.43 ms): opt-in build flag
#endif

#ifndef CM_Z_MINB_D
#define CM_Z_MINB_D 2
#endif
template <typename R, int N> struct ZGeo {
    // 8 elements per thread for power-of-two sides >= 256 so that W and Yh of
    // the whole column fit in registers next to it (prefetched before the
    // forward FFT); other sides keep the y-pass plan
    static constexpr bool E8 = CM_Z_E8 && N >= 256 && (N & (N - 1)) == 0 && sizeof(R) == 4;
    // N >= 512: 16 elements per thread, 16 columns per CTA (128-byte row
    // segments); 512 threads at N = 512 so that two CTAs share an SM (the pass
    // is latency bound: 0.54 -> 0.47 ms at 512^3); W and Yh are then loaded
    // after the forward FFT, in groups of 8
    static constexpr bool E16 = CM_Z_E16 && E8 && N >= CM_Z_E16_MIN;
    static constexpr bool PREFETCH = E8 && !E16;
    // N >= CM_Z_E32_MIN: 32 elements per thread (one warp per column, 512-thread
    // CTAs, up to 128 registers)
    static constexpr bool E32 = E16 && N >= CM_Z_E32_MIN;
    static constexpr int E = E32 ? 32 : E16 ? 16 : E8 ? 8 : Geo<R, N>::EY;
    static constexpr int T = N / E;
    static constexpr int TWMAX = CM_Z_TW ? CM_Z_TW : 16;
    static constexpr int TW = E8 ? (TWMAX < 1024 / T ? TWMAX : 1024 / T) : Geo<R, N>::TWY;
    static constexpr int NT = TW * T;
    static constexpr int NBM = (N / 2 / TW) * N;  // main blocks
    static constexpr size_t SMEM_MAIN0 =
        sizeof(Cx<R>) * (N + (size_t)N * TW) + sizeof(double) * 64 + packed_tw_bytes<R>(N, 2);
    // one GPU, 16-element plan: the CTA's W tile (contiguous in the z-tiled
    // layout) arrives by one cp.async.bulk issued at CTA start, into shared
    // memory next to the exchange buffer; two CTAs per SM still fit
    static constexpr bool WBULK = CM_Z_WBULK && E16 && !E32 && sizeof(R) == 4;
    static constexpr size_t OFF_WB = (SMEM_MAIN0 + 127) / 128 * 128;
    static constexpr size_t SMEM_MAIN = WBULK ? OFF_WB + (size_t)N * TW * 4 + 8 : SMEM_MAIN0;
    // fp64: 16 complex doubles per thread at N >= 512 are 64 registers of data
    // alone; the fp32 bound of 4 CTAs (64 registers) spilled 1.2 KB per thread
    static constexpr int MINB = sizeof(R) == 8 ? CM_Z_MINB_D
                                : (NT >= 1024 || E32) ? 1
                                : E >= 24 ? CM_Z_MINB_E24
                                : (NT <= 256 ? 4 : 2);  // 512 threads: two CTAs per SM
    // column-0 kernel: 8 elements per thread on power-of-two sides >= 256 (more
    // warps per pair block: the kernel is latency bound with 257 blocks)
    static constexpr int E0 = (N >= 256 && (N & (N - 1)) == 0) ? 8 : Geo<R, N>::EY;
    static constexpr int T0 = N / E0;
    static constexpr int NT0 = 2 * T0 < 64 ? 64 : 2 * T0;
    static constexpr size_t SMEM_COL0 =
        sizeof(Cx<R>) * (N + 5 * (size_t)N) + sizeof(double) * 64 + packed_tw_bytes<R>(N, 1);
};

// NR: rows of the spectrum block at compile time (N on one GPU), 0 = p.nrows (b-slab)
template <typename R, int N, int MODE, int NR = N>
__global__ void __launch_bounds__(ZGeo<R, N>::NT, ZGeo<R, N>::MINB) zmain_kernel(ZMParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    constexpr int TW = ZGeo<R, N>::TW, T = ZGeo<R, N>::T, E = ZGeo<R, N>::E, Nh = G::Nh;
    pdl_trigger();
    pdl_wait();
    if (p.st && ld_done(p.st)) {
        // the y-forward pass of the stopping iteration has run; stop the next one
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) p.st->done_y = 1;
        return;
    }
    if constexpr (NR != 0) {
        // L2 prefetch of a later tile (no registers or shared memory held): the
        // pass is latency bound with two CTAs per SM, so the S rows of tile + pf
        // and the z-tiled W / Yh block of tile + pfw are requested ahead
        const int tl = blockIdx.y * gridDim.x + blockIdx.x, ntl = (Nh / ZGeo<R, N>::TW) * NR;
        if (p.pf > 0 && tl + p.pf < ntl && p.tmS) {
            if (threadIdx.x == 0) {
                const int t2 = tl + p.pf, ntx = Nh / ZGeo<R, N>::TW;
                const int hf = 2 * (t2 % ntx) * ZGeo<R, N>::TW, b2 = t2 / ntx;
                for (int c0 = 0; c0 < N; c0 += 256)
                    asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                                     reinterpret_cast<uint64_t>(p.tmS)),
                                 "r"(hf), "r"(b2), "r"(c0)
                                 : "memory");
            }
        } else if (p.pf > 0 && tl + p.pf < ntl) {
            const int t2 = tl + p.pf;
            const Cx<R>* rowp = p.S + (size_t)(t2 / (Nh / ZGeo<R, N>::TW)) * Nh +
                                (t2 % (Nh / ZGeo<R, N>::TW)) * ZGeo<R, N>::TW;
            for (int c = threadIdx.x; c < N; c += blockDim.x)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(rowp + (size_t)c * NR * Nh));
        }
        // (bulk prefetch: 16-byte aligned blocks whose size is a multiple of 16)
        constexpr bool PFW_OK = ((size_t)N * ZGeo<R, N>::TW * sizeof(R)) % 16 == 0;
        if (PFW_OK && MODE != ZM_FWD && p.pfw >= 0 && tl + p.pfw < ntl && threadIdx.x == 0) {
            const size_t o = (size_t)(tl + p.pfw) * N * ZGeo<R, N>::TW;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.W + o),
                         "r"((uint32_t)(N * ZGeo<R, N>::TW * sizeof(R))) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p.Yh + o),
                         "r"((uint32_t)(N * ZGeo<R, N>::TW * sizeof(Cx<R>))) : "memory");
        }
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* buf = tw + N;
    double* red = reinterpret_cast<double*>(buf + N * TW);
    float4* twF = reinterpret_cast<float4*>(red + 64);
    float4* twI = twF + N;
    if constexpr (use_packed_tw<R>()) {
        stage_table(twF, p.twF4, N);
        stage_table(twI, p.twI4, N);
    } else {
        stage_table(tw, p.twN, N);
    }
    const int col = threadIdx.x % TW;
    const int t = threadIdx.x / TW;
    const int nrows = NR ? NR : p.nrows;
    const int hl = NR ? Nh : p.hlen;  // stored row length
    const int h0 = NR ? 0 : p.h0;     // first global column of this launch
    // one (column tile, row b) per CTA: a persistent loop here costs registers
    // (spills at 64 per thread) for less than the twiddle staging it saves
    const int NTX = hl / TW;
    const int tile = blockIdx.y * gridDim.x + blockIdx.x;
    if (tile >= NTX * nrows) return;
    const int hloc = (tile % NTX) * TW + col;
    const int h = h0 + hloc;
    const int b = tile / NTX;  // local row
    const size_t plane = (size_t)nrows * hl;
    C* base = p.S + (size_t)b * hl + hloc;
    constexpr bool WB = ZGeo<R, N>::WBULK && NR != 0 && MODE != ZM_FWD;
    const float* wsm = reinterpret_cast<const float*>(smem_raw + ZGeo<R, N>::OFF_WB);
    const uint32_t wbar = smem_u32(smem_raw + ZGeo<R, N>::OFF_WB + (size_t)N * TW * 4);
    if constexpr (WB) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(wbar));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            mbar_expect_tx_s(wbar, (uint32_t)(N * TW * 4));
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(smem_raw + ZGeo<R, N>::OFF_WB)),
                "l"(reinterpret_cast<uint64_t>(p.W + (size_t)tile * N * TW)), "r"((uint32_t)(N * TW * 4)),
                "r"(wbar)
                : "memory");
        }
    }
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = base[(size_t)(t + T * m) * plane];
    // W and Yh of this column are independent of the transform: with the small
    // plan they are loaded now and land while the forward FFT runs
    R w[E];
    C y[E];
    constexpr bool PREFETCH = ZGeo<R, N>::PREFETCH && MODE != ZM_FWD;
    // W / Yh layout: one GPU (NR = N) stores them z-tiled, [tile][c][TW] with
    // tile = b * NTX + h / TW (convert_acc_kernel), so a CTA's W / Yh tile is
    // one contiguous 32 / 64 KB block instead of 128-byte segments 1 MB apart;
    // b-slab ranks keep [c][b][h]
    auto wy_index = [&](int c) -> size_t {
        if constexpr (NR != 0) return ((size_t)tile * N + c) * TW + col;
        else return ((size_t)c * nrows + b) * hl + hloc;
    };
    if constexpr (PREFETCH) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const size_t gi = wy_index(t + T * m);
            w[m] = __ldg(p.W + gi);
            y[m] = __ldg(p.Yh + gi);
        }
    }
    __syncthreads();
    fft_regs<N, E, N, true>(v, t, buf, ColAddr{TW, col}, tw_src<R, true>(tw, twF), BlockSync{});
    if constexpr (MODE == ZM_FWD) {
        C* const sbase = opaque(base);
        const size_t splane = opaque(plane);
#pragma unroll
        for (int m = 0; m < E; ++m) sbase[(size_t)(t + T * m) * splane] = v[m];
        return;
    }
    // two accumulator pairs (even / odd m): half-length dependency chains
    R quad = R(0), cross = R(0), quad1 = R(0), cross1 = R(0);
    const size_t lplane = opaque(plane);
    if (h == 0) {
#pragma unroll
        for (int m = 0; m < E; ++m) p.Z0[(size_t)b * N + t + T * m] = v[m];
    } else {
        // without the prefetch, W and Yh are consumed in groups of G (a compiler
        // fence between groups bounds the registers held by loads in flight)
        constexpr int G = (PREFETCH || E % 8 != 0) ? E : 8;
#pragma unroll
        for (int g0 = 0; g0 < E; g0 += G) {
            if constexpr (!PREFETCH) {
#pragma unroll
                if (WB && g0 == 0) mbar_wait_s(wbar, 0);  // the W tile landed during the forward FFT
                for (int m = g0; m < g0 + G; ++m) {
                    // b-slab layout through the opaque plane stride (the addresses
                    // are recomputed, not held live: spills at 128 registers)
                    const size_t gi = NR != 0 ? wy_index(t + T * m)
                                              : (size_t)(t + T * m) * lplane + (size_t)b * hl + hloc;
                    w[m] = WB ? wsm[(t + T * m) * TW + col] : __ldg(p.W + gi);
                    y[m] = p.Yh[gi];
                }
            }
#pragma unroll
            for (int m = g0; m < g0 + G; ++m) {
                const C f = v[m];
                // E = 32 (one warp per column at 1024) has no registers to spare
                if ((m & 1) && E <= 16 && NR != 0) {
                    quad1 += w[m] * (f.x * f.x + f.y * f.y);
                    cross1 += y[m].x * f.x + y[m].y * f.y;
                } else {
                    quad += w[m] * (f.x * f.x + f.y * f.y);
                    cross += y[m].x * f.x + y[m].y * f.y;
                }
                v[m] = cx<C>(w[m] * f.x - y[m].x, w[m] * f.y - y[m].y);
            }
            if constexpr (!PREFETCH) asm volatile("" ::: "memory");
        }
    }
    if (p.part) {
        double acc[2] = {2.0 * ((double)quad + (double)quad1),
                         2.0 * ((double)cross + (double)cross1)};  // mates 0 < h < N/2
        block_sum<2>(acc, red);
        if (threadIdx.x == 0) {
            p.part[tile * NP3 + 0] = acc[0];
            p.part[tile * NP3 + 1] = acc[1];
        }
    }
    if constexpr (MODE == ZM_FIT) return;
    __syncthreads();
    fft_regs<N, E, N, false>(v, t, buf, ColAddr{TW, col}, tw_src<R, false>(tw, twI), BlockSync{});
    // recompute the store addresses here instead of holding E 64-bit addresses
    // live across the transforms (register pressure at 64 registers per thread)
    C* const sbase = opaque(base);
    const size_t splane = opaque(plane);
    if (h != 0)
#pragma unroll
        for (int m = 0; m < E; ++m) sbase[(size_t)(t + T * m) * splane] = v[m];
}

template <typename R, int N, int MODE>
__global__ void __launch_bounds__(ZGeo<R, N>::NT0)
zcol0_kernel(ZMParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    constexpr int T = ZGeo<R, N>::T0, E = ZGeo<R, N>::E0, Nh = G::Nh;
    pdl_trigger();
    pdl_wait();
    if (p.st && ld_done(p.st)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* z0s = tw + N;          // [2][N]
    C* bufs = z0s + 2 * N;    // [3][N] (third: scratch of idle threads)
    double* red = reinterpret_cast<double*>(bufs + 3 * N);
    float4* twI = reinterpret_cast<float4*>(red + 64);
    if constexpr (use_packed_tw<R>()) stage_table(twI, p.twI4, N);
    else stage_table(tw, p.twN, N);
    const int bp = blockIdx.x;
    const int r = threadIdx.x / T;             // 0, 1 (and idle threads for tiny N)
    const int t = threadIdx.x % T;
    const int rr = r < 2 ? r : 0;
    const int b = rr == 0 ? bp : (N - bp) % N;
    const bool self = (bp == (N - bp) % N);
    const bool active = (r == 0) || (r == 1 && !self);
    for (int q = threadIdx.x; q < 2 * N; q += blockDim.x) {
        const int rq = q / N, c = q % N;
        const int bq = rq == 0 ? bp : (N - bp) % N;
        z0s[q] = p.Z0[(size_t)bq * N + c];
    }
    __syncthreads();
    const int rm = self ? 0 : 1 - rr;
    C v[E];
    double quad = 0.0, cross = 0.0;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int c = t + T * m;
        const C zz = z0s[rr * N + c];
        const C zm = z0s[rm * N + (N - c) % N];
        // F0 = (Z + conj Zm)/2, FN = (Z - conj Zm)/(2i)
        const C f0 = cx<C>(R(0.5) * (zz.x + zm.x), R(0.5) * (zz.y - zm.y));
        const C fn = cx<C>(R(0.5) * (zz.y + zm.y), R(-0.5) * (zz.x - zm.x));
        const C* q = p.Q0 + ((size_t)b * N + c) * 3;
        const C wq = q[0], y0 = q[1], yn = q[2];
        const R w0 = wq.x, wn = wq.y;
        if (active) {
            quad += (double)w0 * ((double)f0.x * f0.x + (double)f0.y * f0.y) +
                    (double)wn * ((double)fn.x * fn.x + (double)fn.y * fn.y);
            cross += ((double)y0.x * f0.x + (double)y0.y * f0.y) +
                     ((double)yn.x * fn.x + (double)yn.y * fn.y);
        }
        const C g0 = cx<C>(w0 * f0.x - y0.x, w0 * f0.y - y0.y);
        const C gn = cx<C>(wn * fn.x - yn.x, wn * fn.y - yn.y);
        v[m] = cx<C>(g0.x - gn.y, g0.y + gn.x);  // g0 + i gn
    }
    if (p.part) {
        double acc[2] = {quad, cross};
        block_sum<2>(acc, red);
        if (threadIdx.x == 0) {
            const int bid = ZGeo<R, N>::NBM + bp;
            p.part[bid * NP3 + 0] = acc[0];
            p.part[bid * NP3 + 1] = acc[1];
        }
    }
    if constexpr (MODE == ZM_FIT) return;
    __syncthreads();
    fft_regs<N, E, N, false>(v, t, bufs + (r < 2 ? r : 2) * N, ColAddr{1, 0},
                             tw_src<R, false>(tw, twI), BlockSync{});
    if (active && r < 2)
#pragma unroll
        for (int m = 0; m < E; ++m) p.S[((size_t)(t + T * m) * N + b) * Nh] = v[m];
}

} // namespace cm
