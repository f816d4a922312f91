// Fused plane pairs (fp32, one GPU): the y and x transforms of a z plane in ONE
// persistent kernel whose intermediate spectrum stays in L2.
//
//   inverse pair (DIR 0): y inverse of plane p (column tiles)  ->  x C2R of plane p (line groups) -> g
//   forward pair (DIR 1): x R2C of plane p (line groups) -> y forward of plane p (column tiles) -> S
//
// Work items form one global sequence: producer items of plane s, then the
// consumer items of plane s - D (D planes of lag), for s = 0 .. N + D - 1.
// CTA c takes items c, c + G, c + 2G, ... (G CTAs, all co-resident); a consumer
// item waits on a per-plane counter of finished producer items. Producers of an
// item precede it by more than G positions, so the CTA with the smallest
// current item never waits on an unfinished item: no deadlock. With D planes of
// lag consumers rarely wait, and the producer output of the planes in flight
// (~D MB at 512^3) is re-read from L2 instead of HBM. The inverse pair also
// discards the consumed spectrum lines from L2 (discard.global.L2): they are
// dead until the next R2C rewrites them, so they are never written back.
//
// Each CTA prefetches its next item into a shared staging buffer by TMA (2D
// tensor tiles for y column tiles, 1D bulk copies for x line groups) while it
// transforms the current one from registers.
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "tma.cuh"
#include "xfft.cuh"

namespace cm {

template <int N> struct FGeo {
    using G = Geo<float, N>;
    using X = XGeo<float, N>;
    static constexpr int Nh = N / 2;
    static constexpr int TWY = G::TWY, TY = G::TY, EY = G::EY;
    static constexpr int NT = TWY * TY;            // one y column tile per item
    static constexpr int TX = X::T;                // threads per x line
    static constexpr int LG = NT / TX;             // x lines per item
    static constexpr int NYT = Nh / TWY;           // y items per plane
    static constexpr int NXG = N / LG;             // x items per plane
    static constexpr int PER_PLANE = NYT + NXG;
    static constexpr int YBOX = N < 256 ? N : 256; // rows per TMA box
    static constexpr size_t al(size_t v) { return (v + 127) / 128 * 128; }
    static constexpr size_t YIN = 8ull * N * TWY;
    static constexpr size_t XIN0 = 8ull * LG * Nh, XIN1 = 4ull * LG * N;
    static constexpr size_t STG = YIN > XIN0 ? (YIN > XIN1 ? YIN : XIN1) : (XIN0 > XIN1 ? XIN0 : XIN1);
    static constexpr size_t YBUF = 8ull * N * TWY, XBUF = 8ull * LG * X::PADX;
    static constexpr size_t OFF_STG = al(8ull * N);
    static constexpr size_t OFF_BUF = OFF_STG + al(STG);
    static constexpr size_t OFF_BAR = OFF_BUF + al(YBUF > XBUF ? YBUF : XBUF);
    static constexpr size_t SMEM = OFF_BAR + 16;
    static constexpr bool OK = (NT % TX == 0) && (N % LG == 0) && NT <= 1024 && NT >= 32 &&
                               TX <= 32 && N % YBOX == 0 && SMEM <= 227 * 1024;
    static constexpr int MINB = 2 * SMEM <= 227 * 1024 ? 2 : 1;
};

struct FusedParams {
    float2* S;
    float* real;          // inverse: g out (scaled); forward: volume in
    const float2* twN;
    const int* stop;      // &st->done (inverse) / &st->done_y (forward), or null
    int* cnt;             // [N] finished producer items per plane (zeroed before launch)
    float scale;
    int lag;              // D
};

__device__ __forceinline__ void l2_discard(const void* p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <int N, int DIR> struct FusedSeq {
    using F = FGeo<N>;
    static constexpr int NP = DIR == 0 ? F::NYT : F::NXG;  // producers per plane
    static constexpr int NC = DIR == 0 ? F::NXG : F::NYT;  // consumers per plane
    long long head, mid, total;
    int D;
    __device__ __forceinline__ explicit FusedSeq(int lag) : D(lag) {
        head = (long long)D * NP;
        mid = (long long)(N - D) * (NP + NC);
        total = head + mid + (long long)D * NC;
    }
    __device__ __forceinline__ void decode(long long i, bool& prod, int& plane, int& sub) const {
        if (i < head) {
            prod = true;
            plane = (int)(i / NP);
            sub = (int)(i % NP);
        } else if (i < head + mid) {
            const long long r = i - head;
            const int s = D + (int)(r / (NP + NC)), q = (int)(r % (NP + NC));
            prod = q < NP;
            plane = prod ? s : s - D;
            sub = prod ? q : q - NP;
        } else {
            const long long r = i - head - mid;
            prod = false;
            plane = N - D + (int)(r / NC);
            sub = (int)(r % NC);
        }
    }
};

template <int N, int DIR>
__global__ void __launch_bounds__(FGeo<N>::NT, FGeo<N>::MINB)
fused_pair_kernel(FusedParams p, const __grid_constant__ CUtensorMap tmS) {
    using F = FGeo<N>;
    using X = XGeo<float, N>;
    static_assert(F::OK, "fused plane pair: unsupported geometry");
    constexpr int Nh = F::Nh, TWY = F::TWY, TY = F::TY, EY = F::EY, E = X::E, T = X::T;
    if (p.stop && *((volatile const int*)p.stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    float2* tw = reinterpret_cast<float2*>(smem_raw);
    unsigned char* stg = smem_raw + F::OFF_STG;
    float2* buf = reinterpret_cast<float2*>(smem_raw + F::OFF_BUF);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + F::OFF_BAR);
    const int tid = threadIdx.x;
    if (tid == 0) {
        mbar_init(bar, 1);
        mbar_fence_init();
    }
    stage_table(tw, p.twN, N);
    __syncthreads();
    const FusedSeq<N, DIR> seq(p.lag);
    constexpr int NP = FusedSeq<N, DIR>::NP;

    // thread 0: wait for the item's inputs, then start their copy into staging
    auto issue = [&](long long i) {
        bool prod;
        int plane, sub;
        seq.decode(i, prod, plane, sub);
        if (!prod) {
            while (atomicAdd(p.cnt + plane, 0) < NP) __nanosleep(64);
            __threadfence();
            fence_proxy_async();
        }
        if (prod == (DIR == 0)) {  // y column tile: rows plane*N .. +N, columns sub*TWY .. +TWY
            mbar_expect_tx(bar, (uint32_t)F::YIN);
#pragma unroll
            for (int r0 = 0; r0 < N; r0 += F::YBOX)
                tma_load_2d(stg + (size_t)r0 * TWY * 8, &tmS, sub * TWY, plane * N + r0, bar);
        } else if (DIR == 0) {     // C2R input: LG spectrum rows
            mbar_expect_tx(bar, (uint32_t)F::XIN0);
            bulk_load(stg, p.S + ((size_t)plane * N + (size_t)sub * F::LG) * Nh, (uint32_t)F::XIN0, bar);
        } else {                   // R2C input: LG real rows
            mbar_expect_tx(bar, (uint32_t)F::XIN1);
            bulk_load(stg, p.real + ((size_t)plane * N + (size_t)sub * F::LG) * N, (uint32_t)F::XIN1, bar);
        }
    };

    uint32_t phase = 0;
    long long i = blockIdx.x;
    if (tid == 0 && i < seq.total) issue(i);
    for (; i < seq.total; i += gridDim.x) {
        bool prod;
        int plane, sub;
        seq.decode(i, prod, plane, sub);
        mbar_wait(bar, phase);
        phase ^= 1u;
        const bool is_y = prod == (DIR == 0);
        if (is_y) {
            // ---- y transform of a column tile (in place in S)
            const int col = tid % TWY, t = tid / TWY;
            const float2* sv = reinterpret_cast<const float2*>(stg);
            float2 v[EY];
#pragma unroll
            for (int m = 0; m < EY; ++m) v[m] = sv[(t + TY * m) * TWY + col];
            __syncthreads();  // staging consumed
            if (tid == 0 && i + gridDim.x < seq.total) issue(i + gridDim.x);
            fft_regs<N, EY, N, DIR == 1>(v, t, buf, ColAddr{TWY, col},
                                         TwPlain<float2, DIR == 1>{tw}, BlockSync{});
            float2* base = p.S + (size_t)plane * N * Nh + sub * TWY + col;
#pragma unroll
            for (int m = 0; m < EY; ++m) base[(size_t)(t + TY * m) * Nh] = v[m];
        } else {
            // ---- x transforms of LG lines
            const int lg = tid / T, t = tid % T;
            float2* lb = buf + lg * X::PADX;
            const PadAddr pad{};
            const WarpSync wsync{};
            const size_t line = (size_t)plane * N + (size_t)sub * F::LG + lg;
            float2 v[E];
            if constexpr (DIR == 0) {
                // C2R: the mate column Nh - h of the line is in staging too
                const float2* sl = reinterpret_cast<const float2*>(stg) + lg * Nh;
                float2 qm[E];
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = t + T * m;
                    v[m] = sl[hh];
                    qm[m] = sl[(Nh - hh) & (Nh - 1)];
                }
                __syncthreads();
                if (tid == 0 && i + gridDim.x < seq.total) issue(i + gridDim.x);
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = t + T * m;
                    const float2 q = v[m];
                    if (hh == 0) {
                        v[m] = make_float2(q.x + q.y, q.x - q.y);
                    } else {
                        const float2 a = make_float2(q.x + qm[m].x, q.y - qm[m].y);
                        const float2 d = make_float2(q.x - qm[m].x, q.y + qm[m].y);
                        const float2 bb = cmulc(d, tw[hh]);
                        v[m] = make_float2(a.x - bb.y, a.y + bb.x);
                    }
                }
                fft_regs<Nh, E, N, false>(v, t, lb, pad, TwPow<float2, false>{tw}, wsync);
                float* xrow = p.real + line * N;
                const float sc = p.scale;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int pp = t + T * m;
                    *reinterpret_cast<float2*>(xrow + 2 * pp) = make_float2(v[m].x * sc, v[m].y * sc);
                }
            } else {
                const float2* sl = reinterpret_cast<const float2*>(stg) + lg * Nh;  // real pairs
#pragma unroll
                for (int m = 0; m < E; ++m) v[m] = sl[t + T * m];
                __syncthreads();
                if (tid == 0 && i + gridDim.x < seq.total) issue(i + gridDim.x);
                fft_regs<Nh, E, N, true>(v, t, lb, pad, TwPow<float2, true>{tw}, wsync);
                __syncwarp();
#pragma unroll
                for (int m = 0; m < E; ++m) lb[pad(t + T * m)] = v[m];
                __syncwarp();
                float2* Srow = p.S + line * Nh;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int hh = t + T * m;
                    const float2 z = v[m];
                    float2 out;
                    if (hh == 0) {
                        out = make_float2(z.x + z.y, z.x - z.y);
                    } else {
                        const float2 zm = lb[pad(Nh - hh)];
                        const float2 e = make_float2(0.5f * (z.x + zm.x), 0.5f * (z.y - zm.y));
                        const float2 o = make_float2(0.5f * (z.y + zm.y), -0.5f * (z.x - zm.x));
                        out = cadd(e, cmul(o, tw[hh]));
                    }
                    Srow[hh] = out;
                }
            }
        }
        __syncthreads();  // item stored; exchange buffers free
        if (prod) {
            if (tid == 0) {
                __threadfence();
                atomicAdd(p.cnt + plane, 1);
            }
        } else if (DIR == 0) {
            // the consumed spectrum lines are dead until the next R2C rewrites them
            const char* base = reinterpret_cast<const char*>(p.S + ((size_t)plane * N + (size_t)sub * F::LG) * Nh);
            constexpr int NLINES = (int)(F::XIN0 / 128);
            for (int q = tid; q < NLINES; q += blockDim.x) l2_discard(base + (size_t)q * 128);
        }
    }
}

} // namespace cm
