// K3 on sm_100a with TMA — persistent z pass fed by a 2-stage mbarrier ring.
//
// Same mathematics as zmain_kernel (zpass.cuh): FFT along k of TW consecutive
// half-spectrum columns h at one row b, G = W F - Yh with the fit partials
// (regularizer.cpp:91-92, 114-123), inverse FFT along k. The
// tile data moves differently:
//   * one CTA per SM, persistent over tiles (b, h0..h0+TW-1);
//   * thread 0 issues, two tiles ahead, 3D TMA boxes {TW columns, 1 row, 256
//     planes} of S, W and Yh (cp.async.bulk.tensor.3d, mbarrier complete_tx)
//     into a 2-stage shared-memory ring, so the next tile's 80 KB (at 512^3)
//     are in flight while this tile transforms — no registers held for them
//     (the register-prefetch variants of zmain spilled at 64 registers);
//   * the stage's S area doubles as the FFT exchange buffer once the column is
//     in registers; W and Yh are read from shared memory after the forward
//     transform (the multiply does not wait on global memory);
//   * the twiddle table is staged once per CTA, not once per tile;
//   * the fit partials accumulate per CTA in fp64 (fixed tile order:
//     deterministic) and land in part[blockIdx.x]; CTA 0 zeroes the unused
//     zmain slots so the finalize reduction over NBM entries is unchanged.
// Column h = 0 (packed X(0) + i X(N/2)) is left in Z0 for zcol0_kernel, as zmain does.
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "tma.cuh"
#include "zpass.cuh"

namespace cm {

#ifndef CM_ZT_TW
#define CM_ZT_TW 8
#endif

template <int N> struct ZtGeo {
    static constexpr bool OK = (N == 256 || N == 512);
    static constexpr int TW = CM_ZT_TW;                  // columns per tile (64-byte rows)
    static constexpr int E = 8;                          // elements per thread
    static constexpr int T = N / E;                      // threads per column
    static constexpr int NT = TW * T;                    // 512 at N = 512
    static constexpr int Nh = N / 2;
    static constexpr int NTX = Nh / TW;
    static constexpr int NTILES = NTX * N;
    static constexpr int BOXC = N < 256 ? N : 256;       // planes per TMA box (box dims <= 256)
    static constexpr int NBOX = N / BOXC;
    static constexpr uint32_t SB = (uint32_t)N * TW * 8, WB = (uint32_t)N * TW * 4, YB = SB;
    static constexpr size_t OFF_W = SB, OFF_Y = SB + WB, STAGE = SB + WB + YB;
    static constexpr int NSTAGE = 2;
    static constexpr size_t OFF_TW = NSTAGE * STAGE;
    static constexpr size_t OFF_RED = OFF_TW + (size_t)N * 8;
    static constexpr size_t OFF_BAR = OFF_RED + 64 * 8;
    static constexpr size_t SMEM = OFF_BAR + NSTAGE * 8;
    static constexpr int MINB = SMEM * 2 <= 220 * 1024 ? 2 : 1;
};

template <int N, int MODE>
__global__ void __launch_bounds__(ZtGeo<N>::NT, ZtGeo<N>::MINB)
zt_kernel(ZMParams<float> p, const __grid_constant__ CUtensorMap tmS,
          const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmY) {
    using G = ZtGeo<N>;
    using C = float2;
    constexpr int TW = G::TW, E = G::E, T = G::T, NTX = G::NTX, NTILES = G::NTILES;
    constexpr bool WY = MODE != ZM_FWD;
    pdl_trigger();
    pdl_wait();
    if (p.st && ld_done(p.st)) {
        // the y-forward pass of the stopping iteration has run; stop the next one
        if (blockIdx.x == 0 && threadIdx.x == 0) p.st->done_y = 1;
        return;
    }
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw + G::OFF_TW);
    double* red = reinterpret_cast<double*>(smem_raw + G::OFF_RED);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);
    const uint32_t smem_s = smem_u32(smem_raw), bar_s = smem_s + (uint32_t)G::OFF_BAR;
    const int tid = threadIdx.x;
    stage_table(tw, p.twN, N);
    if (tid == 0) {
        for (int s = 0; s < G::NSTAGE; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    if (p.part && blockIdx.x == 0)  // zmain's per-tile slots this kernel does not use
        for (int q = gridDim.x + tid; q < ZGeo<float, N>::NBM; q += blockDim.x) {
            p.part[q * NP3 + 0] = 0.0;
            p.part[q * NP3 + 1] = 0.0;
        }
    __syncthreads();

    auto issue = [&](int tile, int s) {
        const int b = tile / NTX, h0 = (tile % NTX) * TW;
        const uint32_t st = smem_s + (uint32_t)(s * G::STAGE), bs = bar_s + 8u * s;
        mbar_expect_tx_s(bs, G::SB + (WY ? G::WB + G::YB : 0u));
#pragma unroll
        for (int q = 0; q < G::NBOX; ++q) {
            tma_load_3d_s(st + (uint32_t)(q * G::BOXC * TW * 8), &tmS, 2 * h0, b, q * G::BOXC, bs);
            if (WY) {
                tma_load_3d_s(st + (uint32_t)(G::OFF_W + q * G::BOXC * TW * 4), &tmW, h0, b,
                              q * G::BOXC, bs);
                tma_load_3d_s(st + (uint32_t)(G::OFF_Y + q * G::BOXC * TW * 8), &tmY, 2 * h0, b,
                              q * G::BOXC, bs);
            }
        }
    };
    const int stride = gridDim.x;
    if (tid == 0) {
        if ((int)blockIdx.x < NTILES) issue(blockIdx.x, 0);
        if ((int)blockIdx.x + stride < NTILES) issue(blockIdx.x + stride, 1);
    }
    const int col = tid % TW, t = tid / TW;
    const size_t plane = (size_t)N * G::Nh;
    double qsum = 0.0, csum = 0.0;  // thread 0: this CTA's fit partials
    int it = 0;
    for (int tile = blockIdx.x; tile < NTILES; tile += stride, ++it) {
        const int s = it & 1;
        mbar_wait_s(bar_s + 8u * s, (uint32_t)(it >> 1) & 1u);
        C* Ss = reinterpret_cast<C*>(smem_raw + s * G::STAGE);
        const float* Ws = reinterpret_cast<const float*>(smem_raw + s * G::STAGE + G::OFF_W);
        const C* Ys = reinterpret_cast<const C*>(smem_raw + s * G::STAGE + G::OFF_Y);
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = Ss[(t + T * m) * TW + col];
        __syncthreads();  // the S area becomes the exchange buffer
        fft_regs<N, E, N, true>(v, t, Ss, ColAddr{TW, col}, TwPlain<C, true>{tw}, BlockSync{});
        const int b = tile / NTX, h = (tile % NTX) * TW + col;
        C* const gcol = p.S + (size_t)b * G::Nh + h;
        if constexpr (MODE == ZM_FWD) {
#pragma unroll
            for (int m = 0; m < E; ++m) gcol[(size_t)(t + T * m) * plane] = v[m];
        } else {
            float quad = 0.f, cross = 0.f;
            if (h == 0) {
#pragma unroll
                for (int m = 0; m < E; ++m) p.Z0[(size_t)b * N + t + T * m] = v[m];
            } else {
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    const int c = t + T * m;
                    const float w = Ws[c * TW + col];
                    const C y = Ys[c * TW + col];
                    const C f = v[m];
                    quad += w * (f.x * f.x + f.y * f.y);
                    cross += y.x * f.x + y.y * f.y;
                    v[m] = make_float2(w * f.x - y.x, w * f.y - y.y);
                }
            }
            if (p.part) {
                double acc[2] = {2.0 * (double)quad, 2.0 * (double)cross};  // mates 0 < h < N/2
                block_sum<2>(acc, red);
                if (tid == 0) {
                    qsum += acc[0];
                    csum += acc[1];
                }
            }
            if constexpr (MODE == ZM_FULL) {
                fft_regs<N, E, N, false>(v, t, Ss, ColAddr{TW, col}, TwPlain<C, false>{tw},
                                         BlockSync{});
                if (h != 0)
#pragma unroll
                    for (int m = 0; m < E; ++m) gcol[(size_t)(t + T * m) * plane] = v[m];
            }
        }
        // stage s is free: its generic-proxy exchange writes are ordered before the
        // async-proxy (TMA) writes of the tile two ahead
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0 && tile + 2 * stride < NTILES) issue(tile + 2 * stride, s);
    }
    if (p.part && tid == 0) {
        p.part[blockIdx.x * NP3 + 0] = qsum;
        p.part[blockIdx.x * NP3 + 1] = csum;
    }
}

template <int N> inline cudaError_t zt_prepare() {
    cudaError_t e = cudaSuccess;
    for (auto f : {zt_kernel<N, ZM_FULL>, zt_kernel<N, ZM_FIT>, zt_kernel<N, ZM_FWD>})
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)ZtGeo<N>::SMEM);
    return e;
}

// tensor maps of the packed spectrum (S, Yh: float2 rows of Nh) and W (float rows of Nh)
inline int zt_make_map(void* ptr, int N, bool complex_rows, int tw, int boxc, CUtensorMap* out) {
    EncodeTiledFn enc = encode_tiled_fn();
    if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int Nh = N / 2, cw = complex_rows ? 2 : 1;
    const cuuint64_t dims[3] = {(cuuint64_t)cw * Nh, (cuuint64_t)N, (cuuint64_t)N};
    const cuuint64_t strides[2] = {(cuuint64_t)cw * Nh * 4, (cuuint64_t)N * cw * Nh * 4};
    const cuuint32_t box[3] = {(cuuint32_t)(cw * tw), 1, (cuuint32_t)boxc};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CM_ERR_CUDA, "tensor map (z pass) encode failed");
    return CM_OK;
}

} // namespace cm
