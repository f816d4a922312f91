// z-slab distributed M-step solver, fp32, N % 128 == 0.
//
// Rank r of P owns real-space planes k in [r NK, (r+1) NK) (NK = N/P, one ghost
// plane on each side) and, for the z pass, spectrum rows b in [r NB, (r+1) NB)
// (NB = N/P). One iteration on every rank:
//   z pass on its b rows (all c)            zmain_kernel (nrows = NB)
//   all-gather of the packed column-0 pencils, Friedel pairing per row   zcol0r
//   all-to-all  (b-slab -> z-slab)
//   y inverse: destination-major -> natural  ypass_kernel<false, DM>
//   x C2R -> g, stencil sweep (ghost planes), halo exchange of x_{i+1}
//   finalize: local partials -> all-reduce -> audit/trace/tolerance
//   x R2C, y forward: natural -> destination-major (the all-to-all send layout)
//   all-to-all  (z-slab -> b-slab)
// The y passes read/write the destination-major layout [s][k][b_local][h], so
// both transposes are single all-to-alls with no pack/unpack kernels.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "comm.cuh"
#include "impl.cuh"

namespace cm {

// packed column 0 of one local row b (global rb0 + b_local): Friedel pairing
// against the all-gathered pencils, multiply, fit partials, inverse z FFT
template <int N, int MODE>
__global__ void __launch_bounds__(Geo<float, N>::TY < 32 ? 32 : Geo<float, N>::TY)
zcol0r_kernel(ZMParams<float> p, const float2* Z0full, int rb0) {
    using G = Geo<float, N>;
    using C = float2;
    constexpr int T = G::TY, E = G::EY, Nh = G::Nh;
    if (p.st && ld_done(p.st)) return;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    C* tw = reinterpret_cast<C*>(smem_raw);
    C* buf = tw + N;  // [2][N]: the second half is scratch of idle threads (N < 512)
    double* red = reinterpret_cast<double*>(buf + 2 * N);
    stage_table(tw, p.twN, N);
    __syncthreads();
    const int bl = blockIdx.x, b = rb0 + bl, bm = (N - b) % N;
    const int t = threadIdx.x;
    const bool act = t < T;
    C v[E];
    double quad = 0.0, cross = 0.0;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int c = (act ? t : 0) + T * m;
        const C zz = Z0full[(size_t)b * N + c];
        const C zm = Z0full[(size_t)bm * N + (N - c) % N];
        const C f0 = make_float2(0.5f * (zz.x + zm.x), 0.5f * (zz.y - zm.y));
        const C fn = make_float2(0.5f * (zz.y + zm.y), -0.5f * (zz.x - zm.x));
        const C* q = p.Q0 + ((size_t)bl * N + c) * 3;
        const C wq = q[0], y0 = q[1], yn = q[2];
        const float w0 = wq.x, wn = wq.y;
        if (act) {
            quad += (double)w0 * ((double)f0.x * f0.x + (double)f0.y * f0.y) +
                    (double)wn * ((double)fn.x * fn.x + (double)fn.y * fn.y);
            cross += ((double)y0.x * f0.x + (double)y0.y * f0.y) +
                     ((double)yn.x * fn.x + (double)yn.y * fn.y);
        }
        const C g0 = make_float2(w0 * f0.x - y0.x, w0 * f0.y - y0.y);
        const C gn = make_float2(wn * fn.x - yn.x, wn * fn.y - yn.y);
        v[m] = make_float2(g0.x - gn.y, g0.y + gn.x);
    }
    if (p.part) {
        double acc[2] = {quad, cross};
        block_sum<2>(acc, red);
        if (threadIdx.x == 0) {
            const int slot = (Nh / ZGeo<float, N>::TW) * p.nrows + bl;
            p.part[slot * NP3 + 0] = acc[0];
            p.part[slot * NP3 + 1] = acc[1];
        }
    }
    if constexpr (MODE == ZM_FIT) return;
    __syncthreads();
    fft_regs<N, E, N, false>(v, act ? t : 0, buf + (act ? 0 : N), ColAddr{1, 0}, tw, BlockSync{});
    if (act)
#pragma unroll
        for (int m = 0; m < E; ++m) p.S[((size_t)(t + T * m) * p.nrows + bl) * p.hlen] = v[m];
}

// b-slab layout of the packed half spectrum with split column halves:
// [half][c][b_local][h - half N/4], each half one all-to-all (see SpecLayout)
__host__ __device__ inline size_t bslab_index(int n, int nrows, int c, int bl, int a) {
    const int hh = n / 4, half = a >= hh ? 1 : 0;
    return (size_t)half * ((size_t)n * nrows * hh) + ((size_t)c * nrows + bl) * hh + (a - half * hh);
}

// The accumulator rows a rank needs: its b rows [rb0, rb0 + nrows) and their
// Friedel mirrors (N - b) mod N — the projection pairs n with -n. Sorted,
// distinct. 2 nrows rows (fewer when the sets overlap) instead of the N rows
// of the full grid: the upload is 2/P of the 24 N^3 bytes per rank.
inline std::vector<int> acc_rows_needed(int n, int rb0, int nrows) {
    std::vector<char> need(n, 0);
    for (int b = rb0; b < rb0 + nrows; ++b) {
        need[b] = 1;
        need[b ? n - b : 0] = 1;
    }
    std::vector<int> rows;
    for (int b = 0; b < n; ++b)
        if (need[b]) rows.push_back(b);
    return rows;
}

// Sliced fp64 accumulator (W [c][lr][a], Y [c][lr][a] complex over the nrl rows
// of acc_rows_needed; lrow[b] = local row) -> this rank's b rows of the packed
// half spectrum (same projection and sign as convert_acc_kernel).
__global__ static void convert_rows_kernel(int n, int rb0, int nrows, int nrl, const int* __restrict__ lrow,
                                           const double* __restrict__ W, const double* __restrict__ Y,
                                           float* Wm, float* Wn, float2* Ym, float2* Yn, float2* Q0) {
    const int nh = n / 2;
    const size_t total = (size_t)n * nrows * (nh + 1);
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(q % (nh + 1));
        const size_t bc = q / (nh + 1);
        const int bl = (int)(bc % nrows), c = (int)(bc / nrows);
        const int b = rb0 + bl;
        const int am = a ? n - a : 0, bm = b ? n - b : 0, cm_ = c ? n - c : 0;
        const size_t i = ((size_t)c * nrl + lrow[b]) * n + a;
        const size_t m = ((size_t)cm_ * nrl + lrow[bm]) * n + am;
        const double wp = 0.5 * (W[i] + W[m]);
        const double sg = ((a + b + c) & 1) ? -1.0 : 1.0;
        const double pr = sg * 0.5 * (Y[2 * i] + Y[2 * m]), pi = sg * 0.5 * (Y[2 * i + 1] - Y[2 * m + 1]);
        if (a < nh) {
            const size_t o = bslab_index(n, nrows, c, bl, a);
            Wm[o] = float(wp);
            Ym[o] = make_float2(float(pr), float(pi));
        } else {
            const size_t o = (size_t)c * nrows + bl;
            Wn[o] = float(wp);
            Yn[o] = make_float2(float(pr), float(pi));
        }
        if (a == 0 || a == nh) {  // row-major column-0 copy (zcol0r_kernel)
            float2* q = Q0 + ((size_t)bl * n + c) * 3;
            reinterpret_cast<float*>(q)[a == 0 ? 0 : 1] = float(wp);
            q[a == 0 ? 1 : 2] = make_float2(float(pr), float(pi));
        }
    }
}

// Accumulator statistics of one spectrum row b per CTA (the half spectrum's
// (c, a) plane of that row, convert_acc_kernel's terms): out[s * nrows + bl] for
// s = sum W, sum |Z_H|^2, max residue, max scale, max W. The decomposition is
// fixed per row, so the row partials — and their sum in b order on the host —
// do not depend on how many ranks share the rows.
__global__ static void __launch_bounds__(256) acc_row_stats_kernel(int n, int rb0, int nrows, int nrl,
                                                                   const int* __restrict__ lrow,
                                                                   const double* __restrict__ W,
                                                                   const double* __restrict__ Y,
                                                                   double* out) {
    const int nh = n / 2, bl = blockIdx.x, b = rb0 + bl, bm = b ? n - b : 0;
    const size_t lb = (size_t)lrow[b], lm = (size_t)lrow[bm];
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};  // sw, sz, worst, scale, wmax
    const size_t per = (size_t)n * (nh + 1);
    for (size_t q = threadIdx.x; q < per; q += blockDim.x) {
        const int a = (int)(q % (nh + 1)), c = (int)(q / (nh + 1));
        const int am = a ? n - a : 0, cm_ = c ? n - c : 0;
        const size_t i = ((size_t)c * nrl + lb) * n + a, m = ((size_t)cm_ * nrl + lm) * n + am;
        const double w = W[i], wmt = W[m];
        const double yr = Y[2 * i], yi = Y[2 * i + 1], mr = Y[2 * m], mi = Y[2 * m + 1];
        v[2] = fmax(v[2], fmax(hypot(yr - mr, yi + mi), fabs(w - wmt)));
        v[3] = fmax(v[3], fmax(fmax(hypot(yr, yi), w), fmax(hypot(mr, mi), wmt)));
        v[4] = fmax(v[4], fmax(w, wmt));
        const bool inner = (a != 0 && a != nh);
        v[0] += inner ? (w + wmt) : w;
        double zr = 0.0, zi = 0.0;
        if (w > 0.0) {
            const double sc = 1.0 / sqrt(w);
            zr += yr * sc;
            zi += yi * sc;
        }
        if (wmt > 0.0) {
            const double sc = 1.0 / sqrt(wmt);
            zr += mr * sc;
            zi -= mi * sc;
        }
        zr *= 0.5;
        zi *= 0.5;
        v[1] += (inner ? 2.0 : 1.0) * (zr * zr + zi * zi);
    }
    __shared__ double red[8][5];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
        v[1] += __shfl_xor_sync(0xffffffffu, v[1], o);
#pragma unroll
        for (int s = 2; s < 5; ++s) v[s] = fmax(v[s], __shfl_xor_sync(0xffffffffu, v[s], o));
    }
    if (lane == 0)
#pragma unroll
        for (int s = 0; s < 5; ++s) red[wid][s] = v[s];
    __syncthreads();
    if (threadIdx.x == 0) {
        double t[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {  // fixed warp order
            t[0] += red[w][0];
            t[1] += red[w][1];
            for (int s = 2; s < 5; ++s) t[s] = fmax(t[s], red[w][s]);
        }
        for (int s = 0; s < 5; ++s) out[(size_t)s * nrows + bl] = t[s];
    }
}

// w_tv of a frozen weight source on this rank's planes (ghosted layout)
__global__ static void wtv_field_kernel(const float* x, int n, int koff, int nk, float epsp,
                                        float* out) {
    const size_t L = (size_t)n * n * nk;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < L;
         q += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(q % n), j = (int)((q / n) % n), kl = (int)(q / ((size_t)n * n));
        const size_t c = ((size_t)(kl + 1) * n + j) * n + i;
        const float xc = x[c];
        const float d1 = i > 0 ? xc - x[c - 1] : 0.f;
        const float d2 = j > 0 ? xc - x[c - n] : 0.f;
        const float d3 = koff + kl > 0 ? xc - x[c - (size_t)n * n] : 0.f;
        out[c] = 1.f / (sqrtf(d1 * d1 + d2 * d2 + d3 * d3) + epsp);
    }
}

// ---- device-rendered timing problem (1024^3 is rendered on
// the device; the values are a valid Hermitian problem, the cost is data-independent)
__device__ __forceinline__ double hash_unit(unsigned long long seed, unsigned long long i) {
    unsigned long long z = seed * 0x9E3779B97F4A7C15ull + i + 0x632BE59BD9B4E019ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    return (double)(z >> 11) * (1.0 / 9007199254740992.0);
}

// blob lattice (period 24, sigma 3) plus uniform noise; ghost planes included
__global__ static void synth_volume_kernel(int n, int koff, int nk, unsigned long long seed,
                                           float* x, double* sumsq) {
    const size_t NNl = (size_t)n * n;
    const size_t tot = (size_t)(nk + 2) * NNl;
    double acc = 0.0;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < tot;
         q += (size_t)gridDim.x * blockDim.x) {
        const int i = (int)(q % n), j = (int)((q / n) % n), kl = (int)(q / NNl) - 1;
        const int k = koff + kl;
        float v = 0.f;
        if (k >= 0 && k < n) {
            const float di = (float)((i % 24) - 12), dj = (float)((j % 24) - 12),
                        dk = (float)((k % 24) - 12);
            const float r2 = di * di + dj * dj + dk * dk;
            const double u = hash_unit(seed, ((size_t)k * n + j) * n + i);
            v = __expf(-r2 / 18.f) + 0.3f * (float)(u - 0.5);
            if (kl >= 0 && kl < nk) acc += (double)v * v;
        }
        x[q] = v;
    }
    acc = warp_sum(acc);
    if ((threadIdx.x & 31) == 0) atomicAdd(sumsq, acc);
}

// W = 1 + (u(n) + u(-n))/2 on this rank's rows of the packed half spectrum
__global__ static void synth_weight_kernel(int n, int rb0, int nrows, unsigned long long seed,
                                           float* Wm, float* Wn, float2* Q0) {
    const int nh = n / 2;
    const size_t total = (size_t)n * nrows * (nh + 1);
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(q % (nh + 1));
        const size_t bc = q / (nh + 1);
        const int bl = (int)(bc % nrows), c = (int)(bc / nrows);
        const int b = rb0 + bl;
        const int am = a ? n - a : 0, bm = b ? n - b : 0, cm_ = c ? n - c : 0;
        const size_t i = ((size_t)c * n + b) * n + a, m = ((size_t)cm_ * n + bm) * n + am;
        const float w = float(1.0 + 0.5 * (hash_unit(seed ^ 0xABCDull, i) + hash_unit(seed ^ 0xABCDull, m)));
        if (a < nh) Wm[bslab_index(n, nrows, c, bl, a)] = w;
        else Wn[(size_t)c * nrows + bl] = w;
        if (a == 0 || a == nh) reinterpret_cast<float*>(Q0 + ((size_t)bl * n + c) * 3)[a == 0 ? 0 : 1] = w;
    }
}

// Yh = W * F (F: the spectrum of the volume, b-slab layout); packed column and
// Nyquist plane zero (a valid Hermitian choice)
__global__ static void synth_numerator_kernel(size_t count, int hh, size_t half, const float* W,
                                              const float2* F, float2* Yh, float2* Yn, size_t nyq) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < count;
         q += (size_t)gridDim.x * blockDim.x) {
        const float w = W[q];
        const float2 f = F[q];
        const bool col0 = q < half && (q % hh) == 0;  // global column h = 0
        Yh[q] = col0 ? make_float2(0.f, 0.f) : make_float2(w * f.x, w * f.y);
        if (q < nyq) Yn[q] = make_float2(0.f, 0.f);
    }
}

struct DistBase {
    virtual ~DistBase() = default;
    virtual int init() = 0;
    virtual int set_accumulator(const double* w, const double* y, int finalized) = 0;
    virtual int set_volumes(const double* xi, const double* xa) = 0;
    virtual int solve(const cm_reg_config* c, cm_trace_row* tr, int cap, cm_solve_stats* st) = 0;
    virtual int get_volume(double* out) = 0;
    virtual int set_synthetic(unsigned long long seed, double* s_y) = 0;
    std::unique_ptr<Comm> comm;
    int device = 0;
    // accumulator state (full-grid statistics; every rank holds the same values)
    bool acc_set = false, acc_fin = false;
    double residue = 0.0, max_weight = 0.0, s_y = 0.0, s_n = 0.0;
    size_t acc_h2d_bytes = 0;  // host-to-device bytes of the last set_accumulator
};

template <int N>
struct DistImpl final : DistBase {
    using R = float;
    using C = float2;
    static constexpr int Nh = N / 2;
    static constexpr size_t NN = (size_t)N * N;
    using SG = S2Geo<N>;
    using ZG = ZGeo<R, N>;
    using XG = XGeo<R, N>;
    static_assert(N % 128 == 0, "z-slab solver: 128-wide stencil tiles");
    static_assert(!use_packed_tw<R>(), "z-slab kernels use the plain twiddle table");

    struct Rank {
        int r = 0;        // global rank
        int koff = 0;     // first plane
        int rb0 = 0;      // first spectrum row
        R* X[3] = {};
        R* XF[2] = {};
        R* YF[2] = {};
        R* x0keep = nullptr;
        R* anchor = nullptr;
        R* g = nullptr;
        R* wtvf = nullptr;
        C* Snat = nullptr;
        C* Ssend = nullptr;
        C* Srecv = nullptr;
        R* W = nullptr;
        R* Wn = nullptr;
        C* Yh = nullptr;
        C* Yn = nullptr;
        C* Q0 = nullptr;  // [NB][N][3] column-0 inputs, row-major
        C* Z0 = nullptr;
        C* Z0full = nullptr;
        C* twN = nullptr;
        float4* twF4 = nullptr;
        float4* twI4 = nullptr;
        double* part1 = nullptr;
        double* part3 = nullptr;
        double* sums = nullptr;
        DevState* st = nullptr;
        double* trace = nullptr;
        double* theta = nullptr;
        double* rowstat = nullptr;      // [5][NB] accumulator row statistics
        double* rowstat_all = nullptr;  // [P][5][NB] all-gathered
        CUtensorMap tmx[5] = {}, tmp[3] = {}, tmg = {}, tma = {};
    };

    int P = 1, NK = N, NB = N;
    // CM_SLAB_FORCE_COMM=1: run the transposes even on one rank (self send/recv
    // through the communicator; exercises the NCCL all-to-all path on one GPU)
    const bool force_comm = std::getenv("CM_SLAB_FORCE_COMM") != nullptr;
    std::vector<Rank> ranks;
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    double* stage = nullptr;   // fp64 staging (shared by virtual ranks, grown on demand)
    size_t stage_cap = 0;      // doubles
    int* lrow_d = nullptr;     // accumulator row -> staged row (set_accumulator)
    HostXfer xfer;             // pageable host buffers through a pinned ring
    bool vol_set = false, anchor_is_init = false;
    int grid_s2 = 1, grid_x = 1, last_iter = 0, last_fista = 0;
    int ygrid = 1, zgrid = 1;
    bool result_valid = false;
    int trace_cap = 0, theta_cap = 0;

    ~DistImpl() override {
        for (void* p : allocs) cudaFree(p);
        if (stage) cudaFree(stage);
        for (cudaEvent_t e : ev)
            if (e) cudaEventDestroy(e);
        if (cstream) cudaStreamDestroy(cstream);
        if (stream) cudaStreamDestroy(stream);
    }
    template <typename T>
    int dalloc(T** p, size_t count) {
        CK(cudaMalloc((void**)p, sizeof(T) * std::max<size_t>(count, 1)));
        allocs.push_back(*p);
        return CM_OK;
    }
    size_t ghosted() const { return (size_t)(NK + 2) * NN; }

    int map(R* ptr, int zdim, cuuint32_t bw, cuuint32_t bj, CUtensorMap* out) {
        EncodeTiledFn enc = encode_tiled_fn();
        if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)zdim};
        const cuuint64_t strides[2] = {(cuuint64_t)N * 4, (cuuint64_t)NN * 4};
        const cuuint32_t box[3] = {bw, bj, 1};
        const cuuint32_t es[3] = {1, 1, 1};
        if (enc(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
            return fail(CM_ERR_CUDA, "tensor map encode failed");
        return CM_OK;
    }

    int init() override {
        P = comm->P;
        NK = N / P;
        NB = N / P;
        if (N % P != 0 || NK % SG::KC != 0)
            return fail(CM_ERR_INVALID_ARGUMENT, "z-slab decomposition needs N/P a multiple of 64");
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&cstream, cudaStreamNonBlocking));
        for (cudaEvent_t& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        if (Nh % 2 || Hh % ZG::TW || Hh % Geo<R, N>::TWY)
            return fail(CM_ERR_UNSUPPORTED, "z-slab solver: column halves do not tile");
        std::vector<C> tw(N);
        for (int q = 0; q < N; ++q) {
            const double a = -2.0 * M_PI * q / N;
            tw[q] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
        ranks.resize(comm->nv);
        for (int v = 0; v < comm->nv; ++v) {
            Rank& k = ranks[v];
            k.r = comm->rank0 + v;
            k.koff = k.r * NK;
            k.rb0 = k.r * NB;
            for (auto& x : k.X) CKS(dalloc(&x, ghosted()));
            CKS(dalloc(&k.x0keep, ghosted()));
            CKS(dalloc(&k.anchor, ghosted()));
            CKS(dalloc(&k.g, ghosted()));
            const size_t H = (size_t)NK * N * Nh;
            CKS(dalloc(&k.Snat, H));
            CKS(dalloc(&k.Ssend, H));
            if (P > 1 || force_comm) CKS(dalloc(&k.Srecv, H));
            else k.Srecv = k.Ssend;  // one rank: the transposes are the identity
            CKS(dalloc(&k.W, (size_t)N * NB * Nh));
            CKS(dalloc(&k.Wn, (size_t)N * NB));
            CKS(dalloc(&k.Yh, (size_t)N * NB * Nh));
            CKS(dalloc(&k.Yn, (size_t)N * NB));
            CKS(dalloc(&k.Q0, (size_t)3 * N * NB));
            CKS(dalloc(&k.Z0, (size_t)NB * N));
            CKS(dalloc(&k.Z0full, NN));
            CKS(dalloc(&k.twN, N));
            CKS(dalloc(&k.part1, (size_t)std::max(SG::NTILES, 148 * 4) * NP1));
            CKS(dalloc(&k.part3, (size_t)((Nh / ZG::TW) * NB + NB) * NP3));
            CKS(dalloc(&k.sums, NP1 + NP3));
            CKS(dalloc(&k.st, 1));
            for (auto& x : k.X) CK(cudaMemsetAsync(x, 0, ghosted() * 4, stream));
            CK(cudaMemsetAsync(k.g, 0, ghosted() * 4, stream));
            CK(cudaMemcpyAsync(k.twN, tw.data(), sizeof(C) * N, cudaMemcpyHostToDevice, stream));
            for (int q = 0; q < 3; ++q) {
                CKS(map(k.X[q], NK + 2, SG::XW, SG::XR, &k.tmx[q]));
                CKS(map(k.X[q], NK + 2, SG::XW, SG::PR, &k.tmp[q]));
            }
            CKS(map(k.g, NK + 2, SG::CI, SG::TJ, &k.tmg));
            CKS(map(k.anchor, NK + 2, SG::CI, SG::TJ, &k.tma));
        }
        CK(stencil2_prepare<N>());
        CK(cudaFuncSetAttribute(xfft_kernel<R, N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)XG::SMEM));
        CK(cudaFuncSetAttribute(xfft_kernel<R, N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)XG::SMEM));
        CK(cudaFuncSetAttribute(ypass_kernel<R, N, true, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<R, N>::bytes));
        CK(cudaFuncSetAttribute(ypass_kernel<R, N, false, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<R, N>::bytes));
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FULL, 0>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FIT, 0>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FWD, 0>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        int occ = 0, sms = 0;
        CK(stencil2_occupancy<N>(&occ));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const int ntiles = SG::NTI * SG::NTJ * (NK / SG::KC);
        grid_s2 = std::max(1, std::min(ntiles, sms * std::max(occ, 1)));
        int occx = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occx, xfft_kernel<R, N, 0>, XG::NT, XG::SMEM));
        grid_x = sms * std::max(occx, 1);
        int occy = 0, occz = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occy, ypass_kernel<R, N, false, true>,
                                                         Geo<R, N>::TWY * Geo<R, N>::TY,
                                                         YSmem<R, N>::bytes));
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occz, zmain_kernel<R, N, ZM_FULL, 0>,
                                                         ZG::NT, ZG::SMEM_MAIN));
        ygrid = sms * std::max(occy, 1);
        zgrid = sms * std::max(occz, 1);
        CK(cudaStreamSynchronize(stream));
        return CM_OK;
    }

    // ---- data upload ---------------------------------------------------------------
    // fp64 staging, grown on demand: the accumulator rows of one rank (3 nrl N^2
    // doubles) or one rank's ghosted planes of a volume
    int ensure_stage(size_t doubles) {
        if (stage_cap >= doubles) return CM_OK;
        CK(cudaStreamSynchronize(stream));
        if (stage) cudaFree(stage);
        stage = nullptr;
        stage_cap = 0;
        CK(cudaMalloc((void**)&stage, doubles * sizeof(double)));
        stage_cap = doubles;
        return CM_OK;
    }

    // Each rank uploads only the accumulator rows its b-slab conversion reads
    // (acc_rows_needed: its rows and their mirrors), from the caller's pageable
    // arrays through the pinned ring (host_xfer.h); the full-grid statistics
    // are per-row partials (acc_row_stats_kernel) all-gathered across ranks and
    // summed on the host in row order, so every rank — and every P — gets the
    // same numbers.
    int set_accumulator(const double* w, const double* y, int finalized) override {
        if (!lrow_d) CKS(dalloc(&lrow_d, N));
        acc_h2d_bytes = 0;
        std::vector<void*> mine, all;
        for (Rank& k : ranks) {
            if (!k.rowstat) {
                CKS(dalloc(&k.rowstat, 5 * (size_t)NB));
                CKS(dalloc(&k.rowstat_all, 5 * (size_t)N));
            }
            const std::vector<int> rows = acc_rows_needed(N, k.rb0, NB);
            const size_t nrl = rows.size();
            CKS(ensure_stage(3 * nrl * NN));
            std::vector<int> lrow(N, -1);
            for (size_t r = 0; r < nrl; ++r) lrow[rows[r]] = (int)r;
            std::vector<CopySeg> sw, sy;
            for (int c = 0; c < N; ++c)
                for (size_t r = 0; r < nrl;) {
                    size_t e = r + 1;
                    while (e < nrl && rows[e] == rows[e - 1] + 1) ++e;
                    const size_t b0 = (size_t)rows[r], nb = e - r;
                    sw.push_back({w + ((size_t)c * N + b0) * N, nb * N * 8});
                    sy.push_back({y + 2 * (((size_t)c * N + b0) * N), nb * N * 16});
                    r = e;
                }
            double* W = stage;
            double* Y = stage + nrl * NN;
            CKS(xfer.h2d_segments(W, sw, stream));
            CKS(xfer.h2d_segments(Y, sy, stream));
            CK(cudaMemcpyAsync(lrow_d, lrow.data(), sizeof(int) * N, cudaMemcpyHostToDevice, stream));
            acc_h2d_bytes += 24 * nrl * NN;
            acc_row_stats_kernel<<<NB, 256, 0, stream>>>(N, k.rb0, NB, (int)nrl, lrow_d, W, Y, k.rowstat);
            CK(cudaGetLastError());
            convert_rows_kernel<<<grid_for(NN * (Nh + 1) / P, 256), 256, 0, stream>>>(
                N, k.rb0, NB, (int)nrl, lrow_d, W, Y, k.W, k.Wn, k.Yh, k.Yn, k.Q0);
            CK(cudaGetLastError());
            // the stage and the row map are reused by the next hosted rank
            CK(cudaStreamSynchronize(stream));
            mine.push_back(k.rowstat);
            all.push_back(k.rowstat_all);
        }
        if (comm->all_gather(mine, all, sizeof(double) * 5 * NB, stream))
            return fail(CM_ERR_NCCL, "all_gather (accumulator statistics) failed");
        std::vector<double> h(5 * (size_t)N);
        CK(cudaMemcpyAsync(h.data(), ranks[0].rowstat_all, sizeof(double) * h.size(),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double sw = 0.0, sz = 0.0, worst = 0.0, scale = 0.0, wmax = 0.0;
        for (int r = 0; r < P; ++r) {  // rank r holds rows r NB .. r NB + NB - 1: row order
            const double* q = h.data() + (size_t)r * 5 * NB;
            for (int bl = 0; bl < NB; ++bl) {
                sw += q[bl];
                sz += q[NB + bl];
                worst = std::fmax(worst, q[2 * NB + bl]);
                scale = std::fmax(scale, q[3 * NB + bl]);
                wmax = std::fmax(wmax, q[4 * NB + bl]);
            }
        }
        residue = scale > 0.0 ? worst / scale : 0.0;
        max_weight = wmax;
        // scale_data (params.cpp:9-26) by Parseval, as Impl::commit_acc_stage
        const size_t L = NN * N;
        s_n = sw / (double)L;
        s_y = std::sqrt(sz) / (double)L;
        acc_set = true;
        acc_fin = finalized != 0;
        return CM_OK;
    }

    // host full volume -> this rank's ghosted planes (zero outside the grid)
    int upload_slab(const double* host, R* dst, const Rank& k) {
        CKS(ensure_stage(ghosted()));
        CK(cudaMemsetAsync(dst, 0, ghosted() * 4, stream));
        const int k_lo = std::max(0, k.koff - 1), k_hi = std::min(N, k.koff + NK + 1);
        CKS(xfer.h2d(stage, host + (size_t)k_lo * NN, 8 * NN * (k_hi - k_lo), stream));
        const size_t cnt = NN * (k_hi - k_lo);
        to_real_kernel<R><<<grid_for(cnt, 256), 256, 0, stream>>>(
            stage, dst + (size_t)(k_lo - (k.koff - 1)) * NN, cnt);
        CK(cudaGetLastError());
        return CM_OK;
    }

    int set_volumes(const double* xi, const double* xa) override {
        anchor_is_init = xi == xa;
        for (Rank& k : ranks) {
            CKS(upload_slab(xi, k.x0keep, k));
            CKS(upload_slab(xa, k.anchor, k));
        }
        CK(cudaStreamSynchronize(stream));
        vol_set = true;
        return CM_OK;
    }

    // ---- per-phase launches on every local rank ---------------------------------------
    // ---- per-phase launches on every local rank -------------------------------------
    // The spectrum's columns h are split into two halves (Hh = N/4 columns each)
    // stored one after the other in the b-slab (Srecv, W, Yh) and the
    // destination-major (Ssend) layouts, so each half has its own contiguous
    // all-to-all and the transposes of one half overlap the transforms of the
    // other (collectives on `cstream`, ordered by events).
    static constexpr int Hh = Nh / 2;
    size_t half_elems() const { return (size_t)NK * N * Hh; }  // = N * NB * Hh
    SpecLayout nat_layout() const { return spec_layout((long long)N * Nh, 0, N, Nh); }
    SpecLayout dm_layout() const {
        return spec_layout((long long)NB * Hh, (long long)NK * NB * Hh, NB, Hh, (long long)half_elems());
    }
    cudaStream_t cstream = nullptr;  // collectives
    enum Ev { EV_ZA, EV_AG, EV_ZB, EV_C0, EV_IA, EV_IB, EV_ST, EV_HALO, EV_FL, EV_AR, EV_YA, EV_YB,
              EV_FA, EV_FB, EV_N };
    cudaEvent_t ev[EV_N] = {};
    int record(Ev e, cudaStream_t s) {
        CK(cudaEventRecord(ev[e], s));
        return CM_OK;
    }
    int wait(Ev e, cudaStream_t s) {
        CK(cudaStreamWaitEvent(s, ev[e], 0));
        return CM_OK;
    }

    int zmain_half(int half, bool fit_only, bool with_part) {
        for (Rank& k : ranks) {
            const size_t off = (size_t)half * half_elems();
            double* part = with_part ? k.part3 + (size_t)half * (Hh / ZG::TW) * NB * NP3 : nullptr;
            ZMParams<R> p{k.Srecv + off, k.Z0, k.W + off, k.Wn, k.Yh + off, k.Yn, k.twN, k.twF4,
                          k.twI4, part, fit_only ? nullptr : k.st, NB, k.Q0, Hh, half * Hh};
            dim3 grid(Hh / ZG::TW, NB);
            if (fit_only)
                zmain_kernel<R, N, ZM_FIT, 0><<<grid, ZG::NT, ZG::SMEM_MAIN, stream>>>(p);
            else
                zmain_kernel<R, N, ZM_FULL, 0><<<grid, ZG::NT, ZG::SMEM_MAIN, stream>>>(p);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    int gather_col0() {  // on cstream
        std::vector<void*> mine, all;
        for (Rank& k : ranks) {
            mine.push_back(k.Z0);
            all.push_back(k.Z0full);
        }
        if (comm->all_gather(mine, all, sizeof(C) * NB * N, cstream))
            return fail(CM_ERR_NCCL, "all_gather (column 0) failed");
        return CM_OK;
    }
    int zcol0(bool fit_only, bool with_part) {  // column 0 lives in half 0
        const int nt = Geo<R, N>::TY < 32 ? 32 : Geo<R, N>::TY;
        const size_t sm = sizeof(C) * 3 * N + 64 * 8;
        for (Rank& k : ranks) {
            ZMParams<R> p{k.Srecv, k.Z0, k.W, k.Wn, k.Yh, k.Yn, k.twN, k.twF4, k.twI4,
                          with_part ? k.part3 : nullptr, fit_only ? nullptr : k.st, NB, k.Q0, Hh, 0};
            if (fit_only)
                zcol0r_kernel<N, ZM_FIT><<<NB, nt, sm, stream>>>(p, k.Z0full, k.rb0);
            else
                zcol0r_kernel<N, ZM_FULL><<<NB, nt, sm, stream>>>(p, k.Z0full, k.rb0);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    // all-to-all of one column half on cstream; forward: z-slab -> b-slab
    int a2a_half(bool forward, int half) {
        if (P == 1 && !force_comm) return CM_OK;
        std::vector<void*> s, r;
        const size_t off = (size_t)half * half_elems();
        for (Rank& k : ranks) {
            s.push_back((forward ? k.Ssend : k.Srecv) + off);
            r.push_back((forward ? k.Srecv : k.Ssend) + off);
        }
        if (comm->all_to_all(s, r, sizeof(C) * NK * NB * Hh, cstream))
            return fail(CM_ERR_NCCL, "all_to_all failed");
        return CM_OK;
    }
    int y_half(bool fwd, bool use_st, int half) {
        constexpr int TWY = Geo<R, N>::TWY;
        for (Rank& k : ranks) {
            const int* stop = use_st ? (fwd ? &k.st->done_y : &k.st->done) : nullptr;
            YParams<R> p{fwd ? k.Snat : k.Ssend, k.twN, nullptr, stop, fwd ? k.Ssend : k.Snat,
                         fwd ? nat_layout() : dm_layout(), fwd ? dm_layout() : nat_layout(), NK,
                         half * (Hh / TWY), Hh / TWY};
            const int grid = std::min((Hh / TWY) * NK, ygrid);
            if (fwd)
                ypass_kernel<R, N, true, true>
                    <<<grid, TWY * Geo<R, N>::TY, YSmem<R, N>::bytes, stream>>>(p);
            else
                ypass_kernel<R, N, false, true>
                    <<<grid, TWY * Geo<R, N>::TY, YSmem<R, N>::bytes, stream>>>(p);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    // forward transform of the iterate in Snat... -> b-slab Srecv, halves pipelined
    int spectrum_forward(bool use_st) {
        CKS(y_half(true, use_st, 0));
        CKS(record(EV_YA, stream));
        CKS(wait(EV_YA, cstream));
        CKS(a2a_half(true, 0));
        CKS(record(EV_FA, cstream));
        CKS(y_half(true, use_st, 1));
        CKS(record(EV_YB, stream));
        CKS(wait(EV_YB, cstream));
        CKS(a2a_half(true, 1));
        CKS(record(EV_FB, cstream));
        return CM_OK;
    }
    // z pass on both halves + column 0, transposed back to z-slabs, y inverse
    int spectrum_inverse(bool fit_only, bool with_part, bool use_st) {
        CKS(wait(EV_FA, stream));
        CKS(zmain_half(0, fit_only, with_part));
        CKS(record(EV_ZA, stream));
        CKS(wait(EV_ZA, cstream));
        CKS(gather_col0());
        CKS(record(EV_AG, cstream));
        CKS(wait(EV_FB, stream));
        CKS(zmain_half(1, fit_only, with_part));
        CKS(record(EV_ZB, stream));
        CKS(wait(EV_AG, stream));
        CKS(zcol0(fit_only, with_part));
        if (fit_only) return CM_OK;
        CKS(record(EV_C0, stream));
        CKS(wait(EV_C0, cstream));
        CKS(a2a_half(false, 0));
        CKS(record(EV_IA, cstream));
        CKS(a2a_half(false, 1));  // after zmain(B): EV_C0 follows EV_ZB on the compute stream
        CKS(record(EV_IB, cstream));
        CKS(wait(EV_IA, stream));
        CKS(y_half(false, use_st, 0));
        CKS(wait(EV_IB, stream));
        CKS(y_half(false, use_st, 1));
        return CM_OK;
    }
    int x_fft(int dir, std::vector<R*> real, bool use_st) {
        for (size_t v = 0; v < ranks.size(); ++v) {
            Rank& k = ranks[v];
            const int* stop = use_st ? (dir == 0 ? &k.st->done : &k.st->done_y) : nullptr;
            XfParams<R> p{k.Snat, real[v] + NN, k.twN, nullptr, stop, 1.0 / (double)(NN * N),
                          NK * N};
            const int grid = std::min(grid_x, (NK * N + XG::LPC - 1) / XG::LPC);
            if (dir == 0)
                xfft_kernel<R, N, 0><<<grid, XG::NT, XG::SMEM, stream>>>(p);
            else
                xfft_kernel<R, N, 1><<<grid, XG::NT, XG::SMEM, stream>>>(p);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    int halo(std::vector<R*> x) {  // on cstream
        std::vector<void*> lo, hi, glo, ghi;
        for (size_t v = 0; v < ranks.size(); ++v) {
            lo.push_back(x[v] + NN);
            hi.push_back(x[v] + (size_t)NK * NN);
            glo.push_back(x[v]);
            ghi.push_back(x[v] + (size_t)(NK + 1) * NN);
        }
        if (comm->halo(lo, hi, glo, ghi, 4 * NN, cstream)) return fail(CM_ERR_NCCL, "halo failed");
        return CM_OK;
    }
    int finalize(const FinParams& base, bool with_part3, int nb3) {
        for (Rank& k : ranks) {
            fin_local_kernel<<<1, FIN_THREADS, 0, stream>>>(base.part1 ? k.part1 : nullptr, grid_s2,
                                                    with_part3 ? k.part3 : nullptr, nb3, k.sums);
            CK(cudaGetLastError());
        }
        CKS(record(EV_FL, stream));
        CKS(wait(EV_FL, cstream));
        std::vector<double*> sums;
        for (Rank& k : ranks) sums.push_back(k.sums);
        if (comm->all_reduce_sum(sums, NP1 + NP3, cstream))
            return fail(CM_ERR_NCCL, "all_reduce failed");
        CKS(record(EV_AR, cstream));
        CKS(wait(EV_AR, stream));
        for (Rank& k : ranks) {
            FinParams f = base;
            f.st = k.st;
            f.trace = base.trace ? k.trace : nullptr;
            f.sums = k.sums;
            finalize_kernel<<<1, FIN_THREADS, 0, stream>>>(f);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    // both streams drained (end of a solve / before host reads)
    int drain() {
        CK(cudaStreamSynchronize(cstream));
        CK(cudaStreamSynchronize(stream));
        return CM_OK;
    }

    // ---- the solver --------------------------------------------------------------------
    int solve(const cm_reg_config* c, cm_trace_row* trace, int cap, cm_solve_stats* stats) override {
        CKS(validate(c));
        if (!acc_set) return fail(CM_ERR_STATE, "accumulator not set");
        if (!acc_fin || residue > 1e-9)
            return fail(CM_ERR_NON_HERMITIAN, "accumulator is not Friedel-finalized");
        if (!vol_set) return fail(CM_ERR_STATE, "volumes not set");
        const int K = c->inner_iters;
        const bool lipschitz = c->step_rule == 0, fista = c->momentum >= 1;
        const bool convex = c->convex_mode != 0;
        const bool want_trace = trace && cap > 0;
        const bool audit = !fista && (lipschitz || want_trace || c->tol_kind == 1);
        const bool refresh_inner = c->refresh == 0 && !convex;
        const bool wfixed = c->refresh == 1 && !convex;
        if (wfixed && !anchor_is_init)
            return fail(CM_ERR_UNSUPPORTED, "z-slab solver: per_m_step needs x_init == x_anchor");
        const double max_wtv = convex ? 1.0 : 1.0 / c->eps_prime;
        const double lr = lipschitz ? 1.0 / (2.0 * max_weight + 2.0 * c->gamma +
                                             12.0 * c->beta * max_wtv / c->mu)
                                    : c->fixed_step;
        const double slack = c->audit_slack > 0.0 ? c->audit_slack : 1e-6;
        const int tol_kind = (fista && c->tol_kind == 1) ? 2 : c->tol_kind;
        const bool need_part1 = audit || tol_kind == 2 || c->momentum == 2;
        const int nb3 = (Nh / ZG::TW) * NB + NB;
        result_valid = false;

        std::vector<double> th;
        if (fista) {
            th.resize(K + 1);
            double tk = 1.0;
            for (int q = 0; q <= K; ++q) {
                const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tk * tk));
                th[q] = (tk - 1.0) / tn;
                tk = tn;
            }
        }
        const bool grow_theta = fista && theta_cap < K + 1;
        const bool grow_trace = want_trace && trace_cap < K;
        for (Rank& k : ranks) {
            if (fista) {
                for (int q = 0; q < 2; ++q) {
                    if (!k.XF[q]) CKS(dalloc(&k.XF[q], ghosted()));
                    if (!k.YF[q]) {
                        CKS(dalloc(&k.YF[q], ghosted()));
                        CK(cudaMemsetAsync(k.YF[q], 0, ghosted() * 4, stream));
                        CKS(map(k.YF[q], NK + 2, SG::XW, SG::XR, &k.tmx[3 + q]));
                    }
                }
                if (grow_theta) CKS(dalloc(&k.theta, (size_t)K + 1));
                CK(cudaMemcpyAsync(k.theta, th.data(), 8 * (K + 1), cudaMemcpyHostToDevice, stream));
            }
            if (grow_trace) CKS(dalloc(&k.trace, (size_t)K * 15));
            CK(cudaMemcpyAsync(fista ? k.XF[0] : k.X[0], k.x0keep, ghosted() * 4,
                               cudaMemcpyDeviceToDevice, stream));
            if (fista)
                CK(cudaMemcpyAsync(k.YF[0], k.x0keep, ghosted() * 4, cudaMemcpyDeviceToDevice, stream));
            if (wfixed) {
                // frozen weights (regularizer.cpp:178-179): w_tv field of x_init once
                if (!k.wtvf) {
                    CKS(dalloc(&k.wtvf, ghosted()));
                    CK(cudaMemsetAsync(k.wtvf, 0, ghosted() * 4, stream));
                }
                wtv_field_kernel<<<grid_for((size_t)NK * NN, 256), 256, 0, stream>>>(
                    k.anchor, N, k.koff, NK, (float)c->eps_prime, k.wtvf);
                CK(cudaGetLastError());
            }
            DevState hs{};
            hs.max_iters = K;
            hs.diverged_iter = -1;
            hs.audit = audit;
            hs.check_diverge = audit && lipschitz;
            hs.tol_kind = tol_kind;
            hs.fista = fista;
            hs.restart = c->momentum == 2;
            hs.refresh_inner = refresh_inner;
            hs.tol = c->tol;
            hs.audit_slack = slack;
            hs.step = lr;
            CK(cudaMemcpyAsync(k.st, &hs, sizeof(hs), cudaMemcpyHostToDevice, stream));
        }
        if (grow_theta) theta_cap = K + 1;
        if (grow_trace) trace_cap = K;
        if (wfixed) {  // the sweep reads w_tv on the ghost plane above the slab
            std::vector<R*> wv;
            for (Rank& k : ranks) wv.push_back(k.wtvf);
            CKS(record(EV_ST, stream));
            CKS(wait(EV_ST, cstream));
            CKS(halo(wv));
            CKS(record(EV_HALO, cstream));
            CKS(wait(EV_HALO, stream));
        }

        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, stream));

        FinParams fb{};
        fb.nb1 = grid_s2;
        fb.nb3 = nb3;
        fb.alpha = c->alpha;
        fb.beta = c->beta;
        fb.gamma = c->gamma;
        fb.invL = 1.0 / (double)(NN * N);
        auto stencil = [&](int g, bool obj_only) -> int {
            for (Rank& k : ranks) {
                StencilParams<R> p{};
                p.g = k.g;
                p.st = obj_only ? nullptr : k.st;
                p.lr = lr;
                p.alpha = c->alpha;
                p.beta = c->beta;
                p.gamma = c->gamma;
                p.eps = c->eps;
                p.eps_prime = c->eps_prime;
                p.mu = c->mu;
                p.convex = convex;
                p.audit = audit || obj_only;
                p.fista = fista && !obj_only;
                p.trace_full = want_trace;
                p.steptol = tol_kind == 2 && !obj_only;
                p.anchor = k.anchor;
                p.part = (need_part1 || obj_only) ? k.part1 : nullptr;
                p.koff = k.koff;
                p.nk = NK;
                p.zshift = 1;
                p.obj_only = obj_only;
                int xi, pi;
                if (fista) {
                    p.xcur = k.YF[g % 2];
                    p.xold = k.XF[g % 2];
                    p.xnext = k.XF[(g + 1) % 2];
                    p.ynext = k.YF[(g + 1) % 2];
                    p.theta = k.theta;
                    xi = 3 + g % 2;
                    pi = 0;
                } else {
                    p.xcur = k.X[g % 3];
                    p.xnext = k.X[(g + 1) % 3];
                    p.xprev = (p.audit && refresh_inner) ? k.X[(g + 2) % 3] : nullptr;
                    xi = g % 3;
                    pi = (g + 2) % 3;
                }
                if (wfixed) {
                    p.wtvf = k.wtvf;
                    p.wl1src = k.anchor;
                }
                CK(stencil2_launch<N>(p, grid_s2, stream, k.tmx[xi], k.tmp[pi], k.tmg, k.tma));
            }
            return CM_OK;
        };
        // the iterate whose spectrum the next z pass needs (FISTA: y_{k+1})
        auto next_iterate = [&](int g) {
            std::vector<R*> v;
            for (Rank& k : ranks) v.push_back(fista ? k.YF[(g + 1) % 2] : k.X[(g + 1) % 3]);
            return v;
        };
        std::vector<R*> gbufs;
        for (Rank& k : ranks) gbufs.push_back(k.g);

        // spectrum of the starting point
        {
            std::vector<R*> x0;
            for (Rank& k : ranks) x0.push_back(fista ? k.YF[0] : k.X[0]);
            CKS(x_fft(1, x0, false));
            CKS(spectrum_forward(false));
        }
        int launches = 0;
        for (int g = 0; g < K; ++g) {
            // K3 (two column halves) + column 0, transposes, K4 (pipelined)
            CKS(spectrum_inverse(false, audit, true));
            CKS(x_fft(0, gbufs, true));              // K1a: g
            CKS(stencil(g, false));                  // K1b
            const std::vector<R*> nx = next_iterate(g);
            CKS(record(EV_ST, stream));              // ghost planes of the new iterate
            CKS(wait(EV_ST, cstream));               // (overlap the finalize)
            CKS(halo(nx));
            CKS(record(EV_HALO, cstream));
            FinParams f = fb;
            f.part1 = need_part1 ? ranks[0].part1 : nullptr;
            f.trace = want_trace ? ranks[0].trace : nullptr;
            CKS(finalize(f, audit, nb3));            // FIN (local -> all-reduce -> audit)
            CKS(wait(EV_HALO, stream));
            CKS(x_fft(1, nx, true));                 // K1c
            CKS(spectrum_forward(true));             // K2 + z-slab -> b-slab (pipelined)
            launches += 13;
            // every rank holds identical device state after the all-reduce, so
            // every rank takes the same decision from its own copy
            if ((g & 7) == 7 || g == K - 1) {
                int done = 0;
                CK(cudaMemcpyAsync(&done, &ranks[0].st->done, 4, cudaMemcpyDeviceToHost, stream));
                CK(cudaStreamSynchronize(stream));
                if (done) break;
            }
        }
        // the last forward transposes run on cstream
        CKS(wait(EV_FA, stream));
        CKS(wait(EV_FB, stream));
        DevState rs;
        CK(cudaMemcpyAsync(&rs, ranks[0].st, sizeof(rs), cudaMemcpyDeviceToHost, stream));
        CKS(drain());
        if (audit && rs.stop_reason == 1) {
            // close the last trace row (regularizer.cpp:208): fit(x_K) and the
            // penalties of x_K under the weights of iteration K-1
            CKS(spectrum_inverse(true, true, false));
            CKS(stencil(rs.iter, true));
            FinParams f = fb;
            f.part1 = ranks[0].part1;
            f.trace = want_trace ? ranks[0].trace : nullptr;
            f.epilogue = 1;
            CKS(finalize(f, true, nb3));
            launches += 4;
            CK(cudaMemcpyAsync(&rs, ranks[0].st, sizeof(rs), cudaMemcpyDeviceToHost, stream));
        }
        CK(cudaEventRecord(e1, stream));
        CKS(drain());
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        const int rows = std::min(rs.rows, want_trace ? cap : 0);
        if (want_trace && rows > 0) {
            std::vector<double> tr((size_t)rows * 15);
            CK(cudaMemcpy(tr.data(), ranks[0].trace, 8 * tr.size(), cudaMemcpyDeviceToHost));
            for (int r = 0; r < rows; ++r) {
                std::memcpy(trace[r].before, &tr[15 * r], 56);
                std::memcpy(trace[r].after, &tr[15 * r + 7], 56);
                trace[r].step = tr[15 * r + 14];
            }
        }
        last_iter = rs.iter;
        last_fista = fista;
        result_valid = rs.stop_reason != 3;
        if (stats) {
            stats->iterations = rs.iter;
            stats->trace_rows = rows;
            stats->stop_reason = rs.stop_reason;
            stats->diverged_iter = rs.diverged_iter;
            stats->last_rel = rs.last_rel;
            stats->step = lr;
            stats->solve_ms = ms;
            stats->kernel_launches = launches * (int)ranks.size();
        }
        if (rs.stop_reason == 3)
            return fail(CM_ERR_STEP_DIVERGED, "m_step: frozen-weight objective increased");
        return CM_OK;
    }

    int set_synthetic(unsigned long long seed, double* s_y) override {
        double* red = nullptr;
        CKS(dalloc(&red, ranks.size()));
        CK(cudaMemsetAsync(red, 0, 8 * ranks.size(), stream));
        std::vector<R*> xs;
        for (size_t v = 0; v < ranks.size(); ++v) {
            Rank& k = ranks[v];
            synth_volume_kernel<<<grid_for(ghosted(), 256), 256, 0, stream>>>(N, k.koff, NK, seed,
                                                                             k.x0keep, red + v);
            CK(cudaGetLastError());
            CK(cudaMemcpyAsync(k.anchor, k.x0keep, ghosted() * 4, cudaMemcpyDeviceToDevice, stream));
            CK(cudaMemsetAsync(k.Q0, 0, sizeof(C) * 3 * N * NB, stream));  // Y column 0 stays zero
            synth_weight_kernel<<<grid_for((size_t)N * NB * (Nh + 1), 256), 256, 0, stream>>>(
                N, k.rb0, NB, seed, k.W, k.Wn, k.Q0);
            CK(cudaGetLastError());
            xs.push_back(k.x0keep);
        }
        // F = fft3 of the volume through the solver's own transforms
        CKS(x_fft(1, xs, false));
        CKS(spectrum_forward(false));
        CKS(wait(EV_FA, stream));
        CKS(wait(EV_FB, stream));
        for (Rank& k : ranks) {
            for (int half = 0; half < 2; ++half) {
                const size_t off = (size_t)half * half_elems();
                ZMParams<R> p{k.Srecv + off, k.Z0, k.W + off, k.Wn, k.Yh + off, k.Yn, k.twN,
                              nullptr, nullptr, nullptr, nullptr, NB, k.Q0, Hh, half * Hh};
                zmain_kernel<R, N, ZM_FWD, 0>
                    <<<dim3(Hh / ZG::TW, NB), ZG::NT, ZG::SMEM_MAIN, stream>>>(p);
                CK(cudaGetLastError());
            }
            const size_t cnt = (size_t)N * NB * Nh;
            synth_numerator_kernel<<<grid_for(cnt, 256), 256, 0, stream>>>(
                cnt, Hh, half_elems(), k.W, k.Srecv, k.Yh, k.Yn, (size_t)N * NB);
            CK(cudaGetLastError());
        }
        std::vector<double*> rv;
        for (size_t v = 0; v < ranks.size(); ++v) rv.push_back(red + v);
        CKS(record(EV_ST, stream));
        CKS(wait(EV_ST, cstream));
        if (comm->all_reduce_sum(rv, 1, cstream)) return fail(CM_ERR_NCCL, "all_reduce failed");
        CKS(record(EV_AR, cstream));
        CKS(wait(EV_AR, stream));
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, red, 8, cudaMemcpyDeviceToHost, stream));
        CKS(drain());
        cudaFree(red);
        allocs.erase(std::find(allocs.begin(), allocs.end(), (void*)red));
        if (s_y) *s_y = std::sqrt(h / (double)(NN * N));
        residue = 0.0;
        max_weight = 2.0;  // bound of the generator (1 + u, u < 1)
        acc_set = acc_fin = vol_set = anchor_is_init = true;
        return CM_OK;
    }

    // this process's planes of the result into the full host volume
    int get_volume(double* out) override {
        if (!result_valid) return fail(CM_ERR_STATE, "no solver result resident");
        CKS(ensure_stage(ghosted()));
        for (Rank& k : ranks) {
            const R* src = (last_fista ? k.XF[last_iter % 2] : k.X[last_iter % 3]) + NN;
            to_double_kernel<R><<<grid_for((size_t)NK * NN, 256), 256, 0, stream>>>(
                src, stage, (size_t)NK * NN);
            CK(cudaGetLastError());
            CKS(xfer.d2h(out + (size_t)k.koff * NN, stage, 8 * (size_t)NK * NN, stream));
        }
        return CM_OK;
    }
};

} // namespace cm
