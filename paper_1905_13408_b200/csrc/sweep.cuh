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

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"

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
    static constexpr int TJ = largest_divisor_le(N, 8);
    static constexpr int TK = 2;
    static constexpr int LPC = TJ * TK;         // lines per tile
    static constexpr int NT0 = LPC * TX;
    static constexpr int NT = NT0 < 64 ? 64 : NT0;  // threads per CTA
    static constexpr int NW = NT / 32;
    static constexpr int LPCB = NT / TX;        // line buffers (>= LPC; extra groups idle)
    static constexpr int CI = largest_divisor_le(N, 128);  // sweep chunk along x
    static constexpr int PADX = Nh + (Nh >> 3) + 1;
    static constexpr int XSW = CI + 2;                      // staged x row width
    static constexpr int XSR = (TK + 2) * (TJ + 2);         // staged x rows
    static constexpr int XPW = CI + 1;
    static constexpr int XPR = (TK + 1) * (TJ + 1);
    static constexpr int SSW = CI + 1;
    static constexpr int SSR = (TK + 1) * (TJ + 1);
    static constexpr int NTILES = (N / TJ) * (N / TK);
    static constexpr size_t SMEM = sizeof(C) * (N + (size_t)LPCB * PADX) +
                                   sizeof(R) * ((size_t)XSR * XSW + (size_t)XPR * XPW +
                                                (size_t)SSR * SSW) +
                                   sizeof(double) * 32 * NP1;
    static constexpr int MINB = (SMEM * 2 <= 220 * 1024 && NT <= 512) ? 2 : 1;
};

template <typename R> __device__ __forceinline__ R rcp_(R v);
template <> __device__ __forceinline__ float rcp_<float>(float v) { return __frcp_rn(v); }
template <> __device__ __forceinline__ double rcp_<double>(double v) { return 1.0 / v; }
template <typename R> __device__ __forceinline__ R log_(R v);
template <> __device__ __forceinline__ float log_<float>(float v) { return __logf(v); }
template <> __device__ __forceinline__ double log_<double>(double v) { return log(v); }

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
};

template <typename R, int N>
__global__ void __launch_bounds__(SwGeo<R, N>::NT, SwGeo<R, N>::MINB)
sweep_kernel(SweepParams<R> p) {
    using G = SwGeo<R, N>;
    using C = Cx<R>;
    constexpr int Nh = G::Nh, E = G::EX, T = G::TX, TJ = G::TJ, TK = G::TK, LPC = G::LPC;
    constexpr int CI = G::CI, PADX = G::PADX, NT = G::NT, NW = G::NW;
    constexpr int XSW = G::XSW, XPW = G::XPW, SSW = G::SSW;
    if (p.st && ld_done(p.st)) return;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* lines = tw + N;                                        // [LPCB][PADX]
    R* XS = reinterpret_cast<R*>(lines + G::LPCB * PADX);     // [TK+2][TJ+2][CI+2]
    R* XP = XS + G::XSR * XSW;                                // [TK+1][TJ+1][CI+1]
    R* SS = XP + G::XPR * XPW;                                // [TK+1][TJ+1][CI+1]
    double* red = reinterpret_cast<double*>(SS + G::SSR * SSW);
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
    __syncthreads();

    for (int tile = blockIdx.x; tile < G::NTILES; tile += gridDim.x) {
        const int j0 = (tile % (N / TJ)) * TJ;
        const int k0 = (tile / (N / TJ)) * TK;
        // line lg of the tile: (kk, jj) = (lg / TJ, lg % TJ)
        const int my_j = j0 + (lg % TJ), my_k = k0 + (lg / TJ);
        C* Srow = p.S + ((size_t)my_k * N + my_j) * Nh;

        // ---- 1. C2R: G rows -> g (unnormalised) in the line buffers ------------
        {
            C v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) v[m] = fft_active ? Srow[t + T * m] : cx<C>(R(0), R(0));
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

        // ---- 2. sweep in chunks along x -------------------------------------------
        for (int i0 = 0; i0 < N; i0 += CI) {
            // stage x: rows (kk', jj') in [-1, TK] x [-1, TJ], columns [i0-1, i0+CI]
            for (int r = wid; r < G::XSR; r += NW) {
                const int kk = r / (TJ + 2) - 1, jj = r % (TJ + 2) - 1;
                const int gk = k0 + kk, gj = j0 + jj;
                const bool rok = gk >= 0 && gk < N && gj >= 0 && gj < N;
                const R* src = p.xcur + ((size_t)(rok ? gk : 0) * N + (rok ? gj : 0)) * N;
                for (int c = lane; c < XSW; c += 32) {
                    const int gi = i0 - 1 + c;
                    XS[r * XSW + c] = (rok && gi >= 0 && gi < N) ? __ldg(src + gi) : R(0);
                }
            }
            if (p.xprev) {  // rows [-1, TK-1] x [-1, TJ-1], columns [i0-1, i0+CI-1]
                for (int r = wid; r < G::XPR; r += NW) {
                    const int kk = r / (TJ + 1) - 1, jj = r % (TJ + 1) - 1;
                    const int gk = k0 + kk, gj = j0 + jj;
                    const bool rok = gk >= 0 && gj >= 0;
                    const R* src = p.xprev + ((size_t)(rok ? gk : 0) * N + (rok ? gj : 0)) * N;
                    for (int c = lane; c < XPW; c += 32) {
                        const int gi = i0 - 1 + c;
                        XP[r * XPW + c] = (rok && gi >= 0) ? __ldg(src + gi) : R(0);
                    }
                }
            }
            __syncthreads();
            // s on the box (kk, jj, ii) in [0, TK] x [0, TJ] x [0, CI]
            if (has_beta) {
                for (int q = tid; q < G::SSR * SSW; q += NT) {
                    const int ii = q % SSW, r = q / SSW;
                    const int kk = r / (TJ + 1), jj = r % (TJ + 1);
                    const int gi = i0 + ii, gj = j0 + jj, gk = k0 + kk;
                    R sv = R(0);
                    if (gi < N && gj < N && gk < N) {
                        const R* xr = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + (ii + 1);
                        const R xc = xr[0];
                        const R d1 = gi > 0 ? xc - xr[-1] : R(0);
                        const R d2 = gj > 0 ? xc - xr[-XSW] : R(0);
                        const R d3 = gk > 0 ? xc - xr[-(TJ + 2) * XSW] : R(0);
                        const R gn = sqrt(d1 * d1 + d2 * d2 + d3 * d3);
                        R wt = R(1);
                        if (!p.convex)
                            wt = p.wtvf ? __ldg(p.wtvf + ((size_t)gk * N + gj) * N + gi)
                                        : rcp_(gn + epsp);
                        sv = wt * rcp_(mu > gn ? mu : gn);
                    }
                    SS[q] = sv;
                }
            }
            __syncthreads();
            // voxels: warp w -> lines w, w+NW, ...; lane -> x
            // per-chunk partials in R (fp32 in product mode: <= CI/32 * LPC/NW
            // terms per thread), folded into fp64 totals after every chunk
            R fa[NP1];
#pragma unroll
            for (int q = 0; q < NP1; ++q) fa[q] = R(0);
            for (int l = wid; l < LPC; l += NW) {
                const int kk = l / TJ, jj = l % TJ;
                const int gk = k0 + kk, gj = j0 + jj;
                R* lbuf = reinterpret_cast<R*>(lines + l * PADX);
                const size_t rowoff = ((size_t)gk * N + gj) * N;
                for (int ii = lane; ii < CI; ii += 32) {
                    const int gi = i0 + ii;
                    const size_t gidx = rowoff + gi;
                    const R* xr = XS + ((kk + 1) * (TJ + 2) + (jj + 1)) * XSW + (ii + 1);
                    const R xc = xr[0];
                    const R d1 = gi > 0 ? xc - xr[-1] : R(0);
                    const R d2 = gj > 0 ? xc - xr[-XSW] : R(0);
                    const R d3 = gk > 0 ? xc - xr[-(TJ + 2) * XSW] : R(0);
                    const R gn = sqrt(d1 * d1 + d2 * d2 + d3 * d3);
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
                            const R* pr = XP + ((kk + 1) * (TJ + 1) + (jj + 1)) * XPW + (ii + 1);
                            const R pc = pr[0];
                            const R e1 = gi > 0 ? pc - pr[-1] : R(0);
                            const R e2 = gj > 0 ? pc - pr[-XPW] : R(0);
                            const R e3 = gk > 0 ? pc - pr[-(TJ + 1) * XPW] : R(0);
                            const R pl1 = rcp_(fabs(pc) + eps);
                            const R ptv = rcp_(sqrt(e1 * e1 + e2 * e2 + e3 * e3) + epsp);
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
#pragma unroll
            for (int q = 0; q < NP1; ++q) acc[q] += (double)fa[q];
            __syncthreads();
        }

        // ---- 3. R2C of the new iterate (line buffers) -> spectrum rows -------------
        {
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
