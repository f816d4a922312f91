// y forward + z pass + y inverse in ONE persistent kernel, pipelined by column
// group through L2 (fp32, one GPU, N in {256, 512}).
//
// Per iteration the spectrum passes y-forward (end of iteration i), z with the
// Fourier-diagonal data term and y-inverse (start of iteration i+1) touch the
// same 16-column group of the packed spectrum three times: 8H bytes each way
// per pass through HBM when run as separate kernels (60H with W / Yh). Here the
// work is a sequence of items, claimed in order through one atomic counter:
//
//     A(0) A(1) B(0) D  A(2) B(1) C(0)  A(3) B(2) C(1) ...  B(G-1) C(G-2) C(G-1)
//
//   A(g): y-forward tile (plane k, group g)       -- ypass_kernel<true>'s tile
//   B(g): z tile (row b, group g): FFT, G = W F - Yh, fit partials, inverse FFT
//         (zmain_kernel's tile, the z-tiled W / Yh of the same CTA tile)
//   D   : the packed column h = 0 with its Friedel mates (zcol0_kernel), after B(0)
//   C(g): y-inverse tile (plane k, group g)
//
// B(g) waits for all of A(g), D for all of B(0), C(g) for all of B(g) (and C(0)
// for D): per-group completion counters, release (fence + atomic) by the
// finishing CTA, acquire polling by the claiming one. Items are claimed in
// sequence order and only depend on earlier items held by resident CTAs
// (persistent grid), so the waits always end. A group's 32 MB (512^3) is
// written by A, read and rewritten by B and read by C within a few groups'
// time, so those accesses are L2 hits and the intermediate write-backs vanish:
// HBM sees A's reads, W / Yh and C's writes (28H instead of 60H).
// Loads of data produced inside the kernel bypass L1 (ld.global.cg).
// Stop flag: when the solve has stopped (done), only the A items run (the
// y-forward of the stopping iteration) and the last CTA raises done_y.
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "zpass.cuh"

namespace cm {

template <int N> struct YzyGeo {
    using ZG = ZGeo<float, N>;
    using G = Geo<float, N>;
    static constexpr bool OK = (N == 256 || N == 512) && ZG::E == G::EY && ZG::TW == G::TWY &&
                               ZG::NT == G::TWY * G::TY && !use_packed_tw<float>();
    static constexpr int NT = ZG::NT, TW = ZG::TW, E = ZG::E, T = ZG::T, Nh = N / 2;
    static constexpr int NG = Nh / TW;                 // column groups
    static constexpr int NITEMS = 3 * N * NG + N / 2 + 1;
    // counters: [0] claim, [1] finished, [2, 2+NG) A done, [2+NG, 2+2NG) B done, [2+2NG] D done
    static constexpr int NCTR = 3 + 2 * NG;
    static constexpr size_t SMEM_Z = ZG::SMEM_MAIN0, SMEM_D = ZG::SMEM_COL0;
    static constexpr size_t SMEM = SMEM_Z > SMEM_D ? SMEM_Z : SMEM_D;
};

enum YzyItem { YZ_A = 0, YZ_B = 1, YZ_D = 2, YZ_C = 3 };

// the item sequence (host): .x type, .y group, .z index (plane / row / pair)
template <int N> inline std::vector<int4> yzy_items() {
    using Y = YzyGeo<N>;
    std::vector<int4> it;
    it.reserve(Y::NITEMS);
    for (int s = 0; s < Y::NG + 2; ++s) {
        if (s < Y::NG)
            for (int k = 0; k < N; ++k) it.push_back(make_int4(YZ_A, s, k, 0));
        if (s >= 1 && s - 1 < Y::NG)
            for (int b = 0; b < N; ++b) it.push_back(make_int4(YZ_B, s - 1, b, 0));
        if (s == 1)
            for (int bp = 0; bp <= N / 2; ++bp) it.push_back(make_int4(YZ_D, 0, bp, 0));
        if (s >= 2)
            for (int k = 0; k < N; ++k) it.push_back(make_int4(YZ_C, s - 2, k, 0));
    }
    return it;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

template <int N>
__global__ void __launch_bounds__(YzyGeo<N>::NT, 2) yzy_kernel(ZMParams<float> p, const int4* items, int* ctr) {
    using Y = YzyGeo<N>;
    using ZG = ZGeo<float, N>;
    using C = float2;
    constexpr int TW = Y::TW, E = Y::E, T = Y::T, Nh = Y::Nh, NG = Y::NG;
    __shared__ int s_item;
    __shared__ int s_flags;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* buf = tw + N;
    double* red_z = reinterpret_cast<double*>(buf + N * TW);
    C* z0s = tw + N;          // D items: [2][N]
    C* bufs = z0s + 2 * N;    // [3][N]
    double* red_d = reinterpret_cast<double*>(bufs + 3 * N);
    DevState* st = p.st;
    if (threadIdx.x == 0) {
        const int dy = st ? *((volatile const int*)&st->done_y) : 0;
        const int dn = st ? *((volatile const int*)&st->done) : 0;
        s_flags = (dy ? 2 : 0) | (dn ? 1 : 0);
    }
    stage_table(tw, p.twN, N);
    __syncthreads();
    const int flags = s_flags;
    if (flags & 2) return;             // stopped before the last y-forward: nothing to do
    const bool only_a = flags & 1;     // the stopping iteration: its y-forward only
    const int col = threadIdx.x % TW, t = threadIdx.x / TW;
    const size_t plane = (size_t)N * Nh;
    int* const done_a = ctr + 2;
    int* const done_b = ctr + 2 + NG;
    int* const done_d = ctr + 2 + 2 * NG;
    auto wait_for = [&](const int* c, int target) {
        if (threadIdx.x == 0) {
            unsigned ns = 32;
            while (ld_acquire(c) < target) {
                __nanosleep(ns);
                if (ns < 1024) ns *= 2;
            }
        }
        __syncthreads();
    };
    auto release = [&](int* c) {
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(c, 1);
    };
    for (;;) {
        if (threadIdx.x == 0) s_item = atomicAdd(ctr, 1);
        __syncthreads();
        const int q = s_item;
        __syncthreads();  // s_item is rewritten by the next claim
        if (q >= Y::NITEMS) break;
        const int4 it = items[q];
        const int type = it.x, g = it.y, idx = it.z;
        if (only_a && type != YZ_A) {
            if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1) == Y::NITEMS - 1) st->done_y = 1;
            continue;
        }
        if (type == YZ_A || type == YZ_C) {
            if (type == YZ_C) wait_for(g == 0 ? done_d : done_b + g, g == 0 ? N / 2 + 1 : N);
            // y pass tile: plane k = idx, columns g*TW .. g*TW+TW-1 (ypass_kernel)
            C* base = p.S + (size_t)idx * plane + g * TW + col;
            C v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = __ldcg(base + (size_t)(t + T * m) * Nh);
            __syncthreads();
            if (type == YZ_A)
                fft_regs<N, E, N, true>(v, t, buf, ColAddr{TW, col}, TwPlain<C, true>{tw}, BlockSync{});
            else
                fft_regs<N, E, N, false>(v, t, buf, ColAddr{TW, col}, TwPlain<C, false>{tw}, BlockSync{});
#pragma unroll
            for (int m = 0; m < E; ++m) base[(size_t)(t + T * m) * Nh] = v[m];
            if (type == YZ_A) release(done_a + g);
        } else if (type == YZ_B) {
            wait_for(done_a + g, N);
            // z tile: row b = idx, columns g*TW.. (zmain_kernel, one GPU, z-tiled W / Yh)
            const int b = idx, tile = b * NG + g, h = g * TW + col;
            C* base = p.S + (size_t)b * Nh + h;
            C v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = __ldcg(base + (size_t)(t + T * m) * plane);
            __syncthreads();
            fft_regs<N, E, N, true>(v, t, buf, ColAddr{TW, col}, TwPlain<C, true>{tw}, BlockSync{});
            float quad = 0.f, cross = 0.f, quad1 = 0.f, cross1 = 0.f;
            if (h == 0) {
#pragma unroll
                for (int m = 0; m < E; ++m) p.Z0[(size_t)b * N + t + T * m] = v[m];
            } else {
                constexpr int GRP = E % 8 == 0 ? 8 : E;
#pragma unroll
                for (int g0 = 0; g0 < E; g0 += GRP) {
                    float w[GRP];
                    C y[GRP];
#pragma unroll
                    for (int m = 0; m < GRP; ++m) {
                        const size_t gi = ((size_t)tile * N + (t + T * (g0 + m))) * TW + col;
                        w[m] = __ldg(p.W + gi);
                        y[m] = __ldg(p.Yh + gi);
                    }
#pragma unroll
                    for (int m = 0; m < GRP; ++m) {
                        const C f = v[g0 + m];
                        if (m & 1) {
                            quad1 += w[m] * (f.x * f.x + f.y * f.y);
                            cross1 += y[m].x * f.x + y[m].y * f.y;
                        } else {
                            quad += w[m] * (f.x * f.x + f.y * f.y);
                            cross += y[m].x * f.x + y[m].y * f.y;
                        }
                        v[g0 + m] = make_float2(w[m] * f.x - y[m].x, w[m] * f.y - y[m].y);
                    }
                    asm volatile("" ::: "memory");
                }
            }
            if (p.part) {
                double acc[2] = {2.0 * ((double)quad + (double)quad1), 2.0 * ((double)cross + (double)cross1)};
                block_sum<2>(acc, red_z);
                if (threadIdx.x == 0) {
                    p.part[tile * NP3 + 0] = acc[0];
                    p.part[tile * NP3 + 1] = acc[1];
                }
            }
            __syncthreads();
            fft_regs<N, E, N, false>(v, t, buf, ColAddr{TW, col}, TwPlain<C, false>{tw}, BlockSync{});
            if (h != 0)
#pragma unroll
                for (int m = 0; m < E; ++m) base[(size_t)(t + T * m) * plane] = v[m];
            release(done_b + g);
        } else {  // YZ_D: packed column 0 of rows (bp, -bp) (zcol0_kernel)
            wait_for(done_b, N);
            constexpr int T0 = ZG::T0, E0 = ZG::E0;
            const int bp = idx;
            const int r = threadIdx.x / T0, t0 = threadIdx.x % T0;
            const int rr = r < 2 ? r : 0;
            const int b = rr == 0 ? bp : (N - bp) % N;
            const bool self = (bp == (N - bp) % N);
            const bool active = (r == 0) || (r == 1 && !self);
            for (int q2 = threadIdx.x; q2 < 2 * N; q2 += blockDim.x) {
                const int rq = q2 / N, c = q2 % N;
                const int bq = rq == 0 ? bp : (N - bp) % N;
                z0s[q2] = __ldcg(p.Z0 + (size_t)bq * N + c);
            }
            __syncthreads();
            const int rm = self ? 0 : 1 - rr;
            C v[E0];
            double quad = 0.0, cross = 0.0;
#pragma unroll
            for (int m = 0; m < E0; ++m) {
                const int c = t0 + T0 * m;
                const C zz = z0s[rr * N + c];
                const C zm = z0s[rm * N + (N - c) % N];
                const C f0 = make_float2(0.5f * (zz.x + zm.x), 0.5f * (zz.y - zm.y));
                const C fn = make_float2(0.5f * (zz.y + zm.y), -0.5f * (zz.x - zm.x));
                const C* qq = p.Q0 + ((size_t)b * N + c) * 3;
                const C wq = qq[0], y0 = qq[1], yn = qq[2];
                const float w0 = wq.x, wn = wq.y;
                if (active) {
                    quad += (double)w0 * ((double)f0.x * f0.x + (double)f0.y * f0.y) +
                            (double)wn * ((double)fn.x * fn.x + (double)fn.y * fn.y);
                    cross += ((double)y0.x * f0.x + (double)y0.y * f0.y) +
                             ((double)yn.x * fn.x + (double)yn.y * fn.y);
                }
                const C g0v = make_float2(w0 * f0.x - y0.x, w0 * f0.y - y0.y);
                const C gnv = make_float2(wn * fn.x - yn.x, wn * fn.y - yn.y);
                v[m] = make_float2(g0v.x - gnv.y, g0v.y + gnv.x);
            }
            if (p.part) {
                double acc[2] = {quad, cross};
                block_sum<2>(acc, red_d);
                if (threadIdx.x == 0) {
                    const int bid = ZG::NBM + bp;
                    p.part[bid * NP3 + 0] = acc[0];
                    p.part[bid * NP3 + 1] = acc[1];
                }
            }
            __syncthreads();
            // idle threads (r >= 2) transform scratch: each r group its own buffer slot
            C* mybuf = r < 2 ? bufs + r * N : bufs + 2 * N;
            if (r < 3)
                fft_regs<N, E0, N, false>(v, t0, mybuf, ColAddr{1, 0}, TwPlain<C, false>{tw}, BlockSync{});
            else
                fft_regs<N, E0, N, false>(v, t0, bufs + 2 * N, ColAddr{1, 0}, TwPlain<C, false>{tw}, BlockSync{});
            if (active && r < 2)
#pragma unroll
                for (int m = 0; m < E0; ++m) p.S[((size_t)(t0 + T0 * m) * N + b) * Nh] = v[m];
            release(done_d);
        }
        __syncthreads();
        if (threadIdx.x == 0 && atomicAdd(ctr + 1, 1) == Y::NITEMS - 1 && only_a && st) st->done_y = 1;
    }
}

} // namespace cm
