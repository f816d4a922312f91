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
    double* part;   // [nblocks_main + N/2 + 1][NP3]
    DevState* st;
};

template <typename R, int N> struct ZGeo {
    static constexpr int TW = Geo<R, N>::TWY;
    static constexpr int T = Geo<R, N>::TY;
    static constexpr int NT = TW * T;
    static constexpr int NBM = (N / 2 / TW) * N;  // main blocks
    static constexpr size_t SMEM_MAIN = sizeof(Cx<R>) * (N + (size_t)N * TW) + sizeof(double) * 64;
    static constexpr int NT0 = 2 * Geo<R, N>::TY < 64 ? 64 : 2 * Geo<R, N>::TY;
    static constexpr size_t SMEM_COL0 = sizeof(Cx<R>) * (N + 5 * (size_t)N) + sizeof(double) * 64;
};

template <typename R, int N, int MODE>
__global__ void __launch_bounds__(ZGeo<R, N>::NT, 2) zmain_kernel(ZMParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    constexpr int TW = ZGeo<R, N>::TW, T = G::TY, E = G::EY, Nh = G::Nh;
    if (p.st && ld_done(p.st)) {
        // the y-forward pass of the stopping iteration has run; stop the next one
        if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) p.st->done_y = 1;
        return;
    }
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* buf = tw + N;
    double* red = reinterpret_cast<double*>(buf + N * TW);
    stage_table(tw, p.twN, N);
    const int col = threadIdx.x % TW;
    const int t = threadIdx.x / TW;
    const int h = blockIdx.x * TW + col;
    const int b = blockIdx.y;
    const size_t plane = (size_t)N * Nh;
    C* base = p.S + (size_t)b * Nh + h;
    C v[E];
#pragma unroll
    for (int m = 0; m < E; ++m) v[m] = base[(size_t)(t + T * m) * plane];
    __syncthreads();
    fft_regs<N, E, N, true>(v, t, buf, ColAddr{TW, col}, tw, BlockSync{});
    if constexpr (MODE == ZM_FWD) {
#pragma unroll
        for (int m = 0; m < E; ++m) base[(size_t)(t + T * m) * plane] = v[m];
        return;
    }
    R quad = R(0), cross = R(0);
    if (h == 0) {
#pragma unroll
        for (int m = 0; m < E; ++m) p.Z0[(size_t)b * N + t + T * m] = v[m];
    } else {
        // W and Yh of this column: issue every load before the math
        R w[E];
        C y[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const size_t gi = ((size_t)(t + T * m) * N + b) * Nh + h;
            w[m] = __ldg(p.W + gi);
            y[m] = p.Yh[gi];
        }
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const C f = v[m];
            quad += w[m] * (f.x * f.x + f.y * f.y);
            cross += y[m].x * f.x + y[m].y * f.y;
            v[m] = cx<C>(w[m] * f.x - y[m].x, w[m] * f.y - y[m].y);
        }
    }
    if (p.part) {
        double acc[2] = {2.0 * (double)quad, 2.0 * (double)cross};  // mates 0 < h < N/2
        block_sum<2>(acc, red);
        if (threadIdx.x == 0) {
            const int bid = blockIdx.y * gridDim.x + blockIdx.x;
            p.part[bid * NP3 + 0] = acc[0];
            p.part[bid * NP3 + 1] = acc[1];
        }
    }
    if constexpr (MODE == ZM_FIT) return;
    __syncthreads();
    fft_regs<N, E, N, false>(v, t, buf, ColAddr{TW, col}, tw, BlockSync{});
    if (h != 0)
#pragma unroll
        for (int m = 0; m < E; ++m) base[(size_t)(t + T * m) * plane] = v[m];
}

template <typename R, int N, int MODE>
__global__ void __launch_bounds__(2 * Geo<R, N>::TY < 64 ? 64 : 2 * Geo<R, N>::TY)
zcol0_kernel(ZMParams<R> p) {
    using G = Geo<R, N>;
    using C = Cx<R>;
    constexpr int T = G::TY, E = G::EY, Nh = G::Nh;
    if (p.st && ld_done(p.st)) return;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* z0s = tw + N;          // [2][N]
    C* bufs = z0s + 2 * N;    // [3][N] (third: scratch of idle threads)
    double* red = reinterpret_cast<double*>(bufs + 3 * N);
    stage_table(tw, p.twN, N);
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
        const size_t gi = ((size_t)c * N + b) * Nh;
        const size_t ni = (size_t)c * N + b;
        const R w0 = p.W[gi], wn = p.Wn[ni];
        const C y0 = p.Yh[gi], yn = p.Yn[ni];
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
    fft_regs<N, E, N, false>(v, t, bufs + (r < 2 ? r : 2) * N, ColAddr{1, 0}, tw, BlockSync{});
    if (active && r < 2)
#pragma unroll
        for (int m = 0; m < E; ++m) p.S[((size_t)(t + T * m) * N + b) * Nh] = v[m];
}

} // namespace cm
