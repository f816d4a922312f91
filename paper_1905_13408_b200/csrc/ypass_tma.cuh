// K2 / K4 on sm_100a with TMA — persistent y pass fed by a 3-stage mbarrier ring.
//
// Same transform as ypass_kernel (kernels.cuh): for every plane k and column h
// of the packed half spectrum, the length-N FFT along j (rows b), forward
// (K2, after the x R2C) or inverse (K4, after the z pass); part of
// fft3 / ifft3_complex (fourier.cpp:18-31, called from regularizer.cpp:87-101).
// The tile data moves differently:
//   * one tile = TW = 16 consecutive columns (128-byte rows) of one plane k,
//     all N rows; one CTA per SM (two at N = 256), persistent over tiles;
//   * thread 0 issues 3D TMA boxes {16 columns, 256 rows, 1 plane}
//     (cp.async.bulk.tensor.3d, mbarrier complete_tx) NS = 3 tiles ahead into a
//     shared-memory ring: 128 KB of loads in flight per SM at 512^3 without
//     holding a register (the register software pipeline of ypass_kernel caps
//     it at 122 registers and one tile ahead);
//   * 8 elements per thread -> 1024 threads (32 warps) per CTA at N = 512, so
//     the FFT's latency chains are hidden by warps rather than by ILP;
//   * the stage buffer is the FFT exchange buffer once the tile is in
//     registers; results go straight from registers to global memory
//     (coalesced 128-byte row segments).
#pragma once

#include "cm_common.cuh"
#include "fft_engine.cuh"
#include "kernels.cuh"
#include "tma.cuh"

namespace cm {

#ifndef CM_YT_NS
#define CM_YT_NS 3
#endif

template <int N> struct YtGeo {
    static constexpr bool OK = (N == 256 || N == 512);
    static constexpr int TW = 16;                        // columns per tile
    static constexpr int E = 8;                          // elements per thread
    static constexpr int T = N / E;                      // threads per column
    static constexpr int NT = TW * T;                    // 1024 at N = 512
    static constexpr int Nh = N / 2;
    static constexpr int NTX = Nh / TW;
    static constexpr int NTILES = NTX * N;               // (plane, column tile)
    static constexpr int BOXB = N < 256 ? N : 256;       // rows per TMA box (box dims <= 256)
    static constexpr int NBOX = N / BOXB;
    static constexpr uint32_t SB = (uint32_t)N * TW * 8;
    static constexpr int NS = CM_YT_NS;
    static constexpr size_t OFF_TW = (size_t)NS * SB;
    static constexpr size_t OFF_BAR = OFF_TW + (size_t)N * 8;
    static constexpr size_t SMEM = OFF_BAR + NS * 8;
    static constexpr int MINB = (SMEM + 1024) * 2 <= 228 * 1024 ? 2 : 1;
};

template <int N, bool FWD>
__global__ void __launch_bounds__(YtGeo<N>::NT, YtGeo<N>::MINB)
ytma_kernel(float2* S, const float2* twN, const int* stop, const __grid_constant__ CUtensorMap tmS) {
    using G = YtGeo<N>;
    using C = float2;
    constexpr int TW = G::TW, E = G::E, T = G::T, NTX = G::NTX, NTILES = G::NTILES, NS = G::NS;
    pdl_trigger();
    pdl_wait();
    if (stop && *((volatile const int*)stop)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw + G::OFF_TW);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + G::OFF_BAR);
    const uint32_t smem_s = smem_u32(smem_raw), bar_s = smem_s + (uint32_t)G::OFF_BAR;
    const int tid = threadIdx.x;
    stage_table(tw, twN, N);
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bar[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    auto issue = [&](int tile, int s) {
        const int k = tile / NTX, h0 = (tile % NTX) * TW;
        const uint32_t st = smem_s + (uint32_t)(s * G::SB), bs = bar_s + 8u * s;
        mbar_expect_tx_s(bs, G::SB);
#pragma unroll
        for (int q = 0; q < G::NBOX; ++q)
            tma_load_3d_s(st + (uint32_t)(q * G::BOXB * TW * 8), &tmS, 2 * h0, q * G::BOXB, k, bs);
    };
    const int stride = gridDim.x;
    if (tid == 0)
        for (int s = 0; s < NS; ++s)
            if ((int)blockIdx.x + s * stride < NTILES) issue(blockIdx.x + s * stride, s);
    const int col = tid % TW, t = tid / TW;
    int it = 0;
    for (int tile = blockIdx.x; tile < NTILES; tile += stride, ++it) {
        const int s = it % NS;
        mbar_wait_s(bar_s + 8u * s, (uint32_t)(it / NS) & 1u);
        C* Ss = reinterpret_cast<C*>(smem_raw + s * G::SB);
        C v[E];
#pragma unroll
        for (int m = 0; m < E; ++m) v[m] = Ss[(t + T * m) * TW + col];
        __syncthreads();  // the stage becomes the exchange buffer
        fft_regs<N, E, N, FWD>(v, t, Ss, ColAddr{TW, col}, TwPlain<C, FWD>{tw}, BlockSync{});
        const int k = tile / NTX, h = (tile % NTX) * TW + col;
        C* const out = S + (size_t)k * N * G::Nh + h;
#pragma unroll
        for (int m = 0; m < E; ++m) out[(size_t)(t + T * m) * G::Nh] = v[m];
        // the stage's generic-proxy exchange writes before the async-proxy (TMA)
        // writes of the tile NS ahead
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (tid == 0 && tile + NS * stride < NTILES) issue(tile + NS * stride, s);
    }
}

template <int N> inline cudaError_t yt_prepare() {
    cudaError_t e = cudaFuncSetAttribute(ytma_kernel<N, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)YtGeo<N>::SMEM);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(ytma_kernel<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)YtGeo<N>::SMEM);
    return e;
}

// packed spectrum S[k][b][h] (float2, Nh per row) as a 3D float map {2 Nh, N, N}
inline int yt_make_map(void* ptr, int N, int tw, int boxb, CUtensorMap* out, int boxc = 1) {
    EncodeTiledFn enc = encode_tiled_fn();
    if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const int Nh = N / 2;
    const cuuint64_t dims[3] = {(cuuint64_t)2 * Nh, (cuuint64_t)N, (cuuint64_t)N};
    const cuuint64_t strides[2] = {(cuuint64_t)2 * Nh * 4, (cuuint64_t)N * 2 * Nh * 4};
    const cuuint32_t box[3] = {(cuuint32_t)(2 * tw), (cuuint32_t)boxb, (cuuint32_t)boxc};
    const cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(CM_ERR_CUDA, "tensor map (y pass) encode failed");
    return CM_OK;
}

} // namespace cm
