// Host runtime of the B200 M-step solver: one Impl<R, N> per (precision, side).
//
// One context = one GPU, one stream, the accumulator and volumes resident in
// HBM. The iteration loop is captured once per solve as a CUDA graph of six
// iterations (K3 K4 K1 FIN K2 x 6; six = lcm of the 3-buffer ISTA and the
// 2-buffer FISTA rotations) and relaunched; kernels read a device-side stop
// flag so a graph that overshoots the stopping iteration costs only empty
// launches. The host polls that flag with a bounded look-ahead.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/cm_api.h"
#include "finalize.cuh"
#include "kernels.cuh"
#include "stencil.cuh"
#include "stencil2.cuh"
#include "xfft.cuh"
#include "xyfused.cuh"
#include "zpass.cuh"
#include "tma.cuh"
#include "host_xfer.h"

#include <nvtx3/nvToolsExt.h>

namespace cm {

// NVTX range for profilers (nsys / ncu --nvtx): scoped push / pop
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// thread-local last error (defined in cm_api.cu)
int fail(int code, const std::string& msg);

} // namespace cm
#include "ypass_tma.cuh"
#include "k1f.cuh"
#include "yzy.cuh"
namespace cm {

#define CK(call)                                                                         \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess)                                                           \
            return fail(CM_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
    } while (0)

#define CKS(call)                                                                        \
    do {                                                                                 \
        int s_ = (call);                                                                 \
        if (s_ != CM_OK) return s_;                                                      \
    } while (0)

// ---------------------------------------------------------------------------------
// upload / conversion kernels (run once per call, not per iteration)
// ---------------------------------------------------------------------------------
static __device__ __forceinline__ void atomic_max_pos(unsigned long long* a, double v) {
    // non-negative doubles order like their bit patterns
    atomicMax(a, (unsigned long long)__double_as_longlong(v));
}

// Full-grid fp64 accumulator -> packed half spectrum (Hermitian projection,
// (-1)^(a+b+c) sign), symmetry residue (backproject.cpp:103-118), max weight,
// sum weight and the Parseval form of scale_data's whitened RMS.
template <typename R>
__global__ void convert_acc_kernel(int n, const double* __restrict__ W,
                                   const double* __restrict__ Y, R* Wm, R* Wn, Cx<R>* Ym,
                                   Cx<R>* Yn, double* part, unsigned long long* maxes,
                                   Cx<R>* Q0 = nullptr, int ztw = 0) {
    using C = Cx<R>;
    const int nh = n / 2;
    const size_t total = (size_t)n * n * (nh + 1);
    double sw = 0.0, sz = 0.0, worst = 0.0, scale = 0.0, wmax = 0.0;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(q % (nh + 1));
        const size_t bc = q / (nh + 1);
        const int b = (int)(bc % n), c = (int)(bc / n);
        const int am = a ? n - a : 0, bm = b ? n - b : 0, cm_ = c ? n - c : 0;
        const size_t i = ((size_t)c * n + b) * n + a;
        const size_t m = ((size_t)cm_ * n + bm) * n + am;
        const double w = W[i], wmt = W[m];
        const double yr = Y[2 * i], yi = Y[2 * i + 1];
        const double mr = Y[2 * m], mi = Y[2 * m + 1];
        // residue: |Y(n) - conj Y(-n)|, |W(n) - W(-n)|; scale: max |Y|, W
        worst = fmax(worst, hypot(yr - mr, yi + mi));
        worst = fmax(worst, fabs(w - wmt));
        scale = fmax(scale, fmax(hypot(yr, yi), w));
        scale = fmax(scale, fmax(hypot(mr, mi), wmt));
        wmax = fmax(wmax, fmax(w, wmt));
        const bool inner = (a != 0 && a != nh);
        sw += inner ? (w + wmt) : w;
        // whitened Hermitian part Z_H = (Y/sqrtW + conj(Ym/sqrtWm)) / 2
        double zr = 0.0, zi = 0.0;
        if (w > 0.0) {
            const double s = 1.0 / sqrt(w);
            zr += yr * s;
            zi += yi * s;
        }
        if (wmt > 0.0) {
            const double s = 1.0 / sqrt(wmt);
            zr += mr * s;
            zi -= mi * s;
        }
        zr *= 0.5;
        zi *= 0.5;
        sz += (inner ? 2.0 : 1.0) * (zr * zr + zi * zi);
        // projected, sign-folded solver inputs
        const double wp = 0.5 * (w + wmt);
        const double sg = ((a + b + c) & 1) ? -1.0 : 1.0;
        const double pr = sg * 0.5 * (yr + mr), pi = sg * 0.5 * (yi - mi);
        if (!Wm) {  // statistics only (z-slab ranks convert their own rows)
        } else if (a < nh) {
            // ztw > 0: z-tiled [b * nh/ztw + a/ztw][c][ztw] (zmain_kernel's W / Yh tiles)
            const size_t o = ztw ? (((size_t)b * (nh / ztw) + a / ztw) * n + c) * ztw + a % ztw
                                 : ((size_t)c * n + b) * nh + a;
            Wm[o] = R(wp);
            Ym[o] = cx<C>(R(pr), R(pi));
        } else {
            const size_t o = (size_t)c * n + b;
            Wn[o] = R(wp);
            Yn[o] = cx<C>(R(pr), R(pi));
        }
        if (Q0 && (a == 0 || a == nh)) {  // row-major column-0 copy (zcol0_kernel)
            C* q = Q0 + ((size_t)b * n + c) * 3;
            R* wq = reinterpret_cast<R*>(q);
            wq[a == 0 ? 0 : 1] = R(wp);
            q[a == 0 ? 1 : 2] = cx<C>(R(pr), R(pi));
        }
    }
    __shared__ double red[32 * 2];
    double v[2] = {sw, sz};
    block_sum<2>(v, red);
    if (threadIdx.x == 0) {
        part[blockIdx.x * 2 + 0] = v[0];
        part[blockIdx.x * 2 + 1] = v[1];
    }
    // maxima: warp-reduce then one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
        worst = fmax(worst, __shfl_xor_sync(0xffffffffu, worst, o));
        scale = fmax(scale, __shfl_xor_sync(0xffffffffu, scale, o));
        wmax = fmax(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    }
    if ((threadIdx.x & 31) == 0) {
        atomic_max_pos(maxes + 0, worst);
        atomic_max_pos(maxes + 1, scale);
        atomic_max_pos(maxes + 2, wmax);
    }
}

template <typename R>
__global__ void to_real_kernel(const double* __restrict__ in, R* __restrict__ out, size_t L) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < L;
         q += (size_t)gridDim.x * blockDim.x)
        out[q] = R(in[q]);
}

// MRC payloads (mode 2 float32) <-> the working precision
template <typename R>
__global__ void f32_to_real_kernel(const float* __restrict__ in, R* __restrict__ out, size_t L) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < L;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = (R)in[i];
}
template <typename R>
__global__ void real_to_f32_kernel(const R* __restrict__ in, float* __restrict__ out, size_t L) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < L;
         i += (size_t)gridDim.x * blockDim.x)
        out[i] = (float)in[i];  // round to nearest, as float(double) in write_mrc
}

template <typename R>
__global__ void to_double_kernel(const R* __restrict__ in, double* __restrict__ out, size_t L) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < L;
         q += (size_t)gridDim.x * blockDim.x)
        out[q] = double(in[q]);
}

// Packed half spectrum (after the x R2C and the y, z forward passes: fft3 of
// the volume) -> full complex fp64 grid, x fastest (fourier.hpp:6-9 layout);
// centered: times (-1)^(a+b+c), i.e. fft3_centered (fourier.cpp:109)
template <typename R>
__global__ void unpack_full_kernel(int n, const Cx<R>* __restrict__ S, double* __restrict__ out,
                                   int centered) {
    const int nh = n / 2;
    const size_t total = (size_t)n * n * n;
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(q % n);
        const size_t bc = q / n;
        const int b = (int)(bc % n), c = (int)(bc / n);
        const int bm = b ? n - b : 0, cm_ = c ? n - c : 0;
        double re, im;
        if (a > 0 && a < nh) {
            const Cx<R> z = S[((size_t)c * n + b) * nh + a];
            re = z.x;
            im = z.y;
        } else if (a > nh) {  // Friedel mate of (n - a, -b, -c)
            const Cx<R> z = S[((size_t)cm_ * n + bm) * nh + (n - a)];
            re = z.x;
            im = -(double)z.y;
        } else {  // column 0 carries F(0) + i F(n/2): separate with the mate
            const Cx<R> z = S[((size_t)c * n + b) * nh], zm = S[((size_t)cm_ * n + bm) * nh];
            if (a == 0) {
                re = 0.5 * ((double)z.x + zm.x);
                im = 0.5 * ((double)z.y - zm.y);
            } else {
                re = 0.5 * ((double)z.y + zm.y);
                im = -0.5 * ((double)z.x - zm.x);
            }
        }
        const double sg = (centered && ((a + b + c) & 1)) ? -1.0 : 1.0;
        out[2 * q] = sg * re;
        out[2 * q + 1] = sg * im;
    }
}

// FSC shell sums (fsc.cpp:10-42) of two packed half spectra of real volumes:
// per shell r = round(|(h, k, l)|) <= n/2: Re sum x conj(y), sum |x|^2, sum |y|^2
// over the full grid (columns 0 < h < n/2 stand for their Friedel mates too,
// weight 2; the packed column 0 is split into h = 0 and h = n/2). The centring
// sign of fft3_centered cancels in every sum. Per-block shared histograms
// (fp64 shared atomics), then a fixed-order sum over blocks.
template <typename R>
__global__ void fsc_shell_kernel(int n, const Cx<R>* __restrict__ Sa, const Cx<R>* __restrict__ Sb,
                                 double* __restrict__ part) {
    extern __shared__ double hist[];  // [n/2 + 1][3]
    const int nh = n / 2, ns = nh + 1;
    for (int q = threadIdx.x; q < 3 * ns; q += blockDim.x) hist[q] = 0.0;
    __syncthreads();
    const size_t total = (size_t)n * n * nh;
    auto add = [&](int h, int k, int l, double xr, double xi, double yr, double yi, double wgt) {
        const int r = (int)lround(sqrt((double)h * h + (double)k * k + (double)l * l));
        if (r > nh) return;
        atomicAdd(&hist[3 * r + 0], wgt * (xr * yr + xi * yi));
        atomicAdd(&hist[3 * r + 1], wgt * (xr * xr + xi * xi));
        atomicAdd(&hist[3 * r + 2], wgt * (yr * yr + yi * yi));
    };
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < total;
         q += (size_t)gridDim.x * blockDim.x) {
        const int a = (int)(q % nh);
        const size_t bc = q / nh;
        const int b = (int)(bc % n), c = (int)(bc / n);
        const int k = b < nh ? b : b - n, l = c < nh ? c : c - n;
        const Cx<R> x = Sa[q], y = Sb[q];
        if (a > 0) {
            add(a, k, l, x.x, x.y, y.x, y.y, 2.0);
        } else {
            const int bm = b ? n - b : 0, cm_ = c ? n - c : 0;
            const size_t m = ((size_t)cm_ * n + bm) * nh;
            const Cx<R> xm = Sa[m], ym = Sb[m];
            // F(0) = (z + conj zm)/2, F(n/2) = (z - conj zm)/(2i)
            add(0, k, l, 0.5 * ((double)x.x + xm.x), 0.5 * ((double)x.y - xm.y),
                0.5 * ((double)y.x + ym.x), 0.5 * ((double)y.y - ym.y), 1.0);
            add(nh, k, l, 0.5 * ((double)x.y + xm.y), -0.5 * ((double)x.x - xm.x),
                0.5 * ((double)y.y + ym.y), -0.5 * ((double)y.x - ym.x), 1.0);
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < 3 * ns; q += blockDim.x)
        part[(size_t)blockIdx.x * 3 * ns + q] = hist[q];
}

__global__ static void fsc_reduce_kernel(const double* __restrict__ part, int nblocks, int len,
                                         double* __restrict__ out) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < len; q += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int b = 0; b < nblocks; ++b) s += part[(size_t)b * len + q];  // fixed order
        out[q] = s;
    }
}

// prox_l1 (regularizer.cpp:103-110), elementwise in fp64
static __global__ void prox_kernel(const double* __restrict__ x, const double* __restrict__ t,
                            double* __restrict__ out, size_t L) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < L;
         q += (size_t)gridDim.x * blockDim.x) {
        const double v = x[q], th = t[q];
        out[q] = fabs(v) <= th ? 0.0 : v - copysign(th, v);
    }
}

inline int grid_for(size_t work, int block) {
    size_t g = (work + block - 1) / block;
    return (int)std::min<size_t>(g, 148 * 32);
}

// ---------------------------------------------------------------------------------
// validation mirrors validate_reg_config (regularizer.cpp:33-42)
// ---------------------------------------------------------------------------------
inline int validate(const cm_reg_config* c) {
    if (!c) return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: null config");
    if (c->alpha < 0.0 || c->beta < 0.0 || c->gamma < 0.0)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: alpha/beta/gamma must be >= 0");
    if (c->eps <= 0.0 || c->eps_prime <= 0.0 || c->mu <= 0.0)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: eps/eps_prime/mu must be > 0");
    if (c->inner_iters < 1)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: inner_iters must be >= 1");
    if (c->step_rule == 1 && c->fixed_step <= 0.0)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: fixed step must be > 0");
    if (c->step_rule != 0 && c->step_rule != 1)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: unknown step rule");
    if (c->refresh != 0 && c->refresh != 1)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: unknown refresh mode");
    if (c->momentum < 0 || c->momentum > 2)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: unknown momentum mode");
    if (c->tol_kind < 0 || c->tol_kind > 2)
        return fail(CM_ERR_INVALID_ARGUMENT, "regularizer: unknown tolerance kind");
    return CM_OK;
}

// ---------------------------------------------------------------------------------
struct ImplBase {
    virtual ~ImplBase() = default;
    virtual int init() = 0;
    virtual int set_accumulator(const double* w, const double* y, int finalized) = 0;
    virtual int set_volumes(const double* xi, const double* xa) = 0;
    virtual int solve(const cm_reg_config* c, cm_trace_row* tr, int cap, cm_solve_stats* st) = 0;
    virtual int get_volume(double* out) = 0;
    virtual int data_gradient(const double* x, double* out) = 0;
    virtual int weights(const double* x, double eps, double epsp, int convex, double* wl1,
                        double* wtv) = 0;
    virtual int tv(const double* x, double mu, const double* wtv, double* value,
                   double* grad) = 0;
    virtual int prox(const double* x, const double* t, double* out) = 0;
    virtual int objective(const double* x, const cm_reg_config* c, const double* anchor,
                          const double* wsrc, double* out7) = 0;
    virtual int fft3(const double* x, double* out, int centered = 0) = 0;
    // fft3_centered of the resident solve result (em_refine, refine.cpp:182)
    virtual int result_spectrum(double* out, int centered) = 0;
    // FSC of this context's and another's resident results (refine.cpp:194)
    virtual int fsc_with(ImplBase* other, double* curve) = 0;
    virtual int result_to_spectrum() = 0;  // S <- fft3 of the resident result
    virtual long long bytes() const = 0;
    // MRC I/O (cm_api.cu): float32 payload landing zone of volume `which`
    // (0 init, 1 anchor) -- the volume itself in fp32, a staging area in fp64 --
    // then mrc_commit(which) (stream-ordered conversion; which 2: anchor = init)
    virtual float* mrc_landing(int which) = 0;
    virtual int mrc_commit(int which) = 0;
    // the resident result as float32 on the device (stream-ordered), or null
    virtual const float* mrc_result_f32() = 0;
    // accumulator staging (3L doubles: weight, numerator interleaved) and its
    // conversion to the resident W / Y (backproject.cuh writes it on the device)
    virtual double* acc_stage() = 0;
    virtual int commit_acc_stage(int finalized) = 0;
    // fft3(_centered) of the resident result as a full fp64 grid in the staging
    // buffer (stream-ordered; estep.cuh reads V from it), or null
    virtual const double* result_spectrum_device(int centered) = 0;

    cudaStream_t stream = nullptr;
    HostXfer xfer;  // pinned chunk ring for the drop-in's pageable host buffers
    int n = 0;
    bool acc_set = false, acc_finalized = false, vol_set = false, anchor_is_init = false;
    double residue = 0.0, max_weight = 0.0, s_y = 0.0, s_n = 0.0;
    int profiling = 0;      // per-kernel CUDA-event timing (no graph)
    double prof_ms[8] = {}; // zmain+zcol0, y-inv, x-C2R, stencil, FIN, x-R2C, y-fwd (ms)
    int prof_iters = 0;
    int last_iter = 0;      // iterations behind the resident result
    int last_fista = 0;
    bool result_valid = false;
};

template <typename R, int N>
struct Impl final : ImplBase {
    using C = Cx<R>;
    using G = Geo<R, N>;
    static constexpr size_t L = (size_t)N * N * N;
    static constexpr int Nh = N / 2;
    static constexpr size_t H = (size_t)N * N * Nh;
    static constexpr size_t NN = (size_t)N * N;
    static constexpr int NB1 = (int)((NN + G::LPC - 1) / G::LPC);
    static constexpr int NB3 = ZGeo<R, N>::NBM + N / 2 + 1;
    static constexpr int LOOK = 8;

    R* X[3] = {};
    R* XF[2] = {};
    R* YF[2] = {};
    R* x0keep = nullptr;
    R* anchor = nullptr;
    R* winit = nullptr;
    R* wtvf = nullptr;         // per_m_step w_tv field (constant within a solve)
    R* gbuf = nullptr;         // data gradient in real space (x-line C2R output)
    CUtensorMap tm_x[5] = {};  // TMA x-box maps of X[0..2], YF[0..1] (fp32 stencil)
    CUtensorMap tm_p[3] = {};  // x_prev boxes of X[0..2]
    CUtensorMap tm_gt = {};    // g tiles
    CUtensorMap tm_at = {};    // anchor tiles
    // z-marching stencil (fp32, N >= 128, N % 8 == 0; the last 128-wide x tile
    // partial when 128 does not divide N): per-plane slab maps
    // z-marching sweep (stencil2.cuh): fp32, and the fp64 parity mode (2 voxels per lane)
    static constexpr bool S2 = N >= 128 && N % 8 == 0;
    CUtensorMap tm2_x[5] = {}, tm2_p[3] = {}, tm2_g = {}, tm2_a = {};
    int s2_grid = 0;
    int sweep_grid = 0;        // persistent stencil CTAs
    int xfft_grid = 0;         // persistent x-line transform CTAs
    int ygrid = 1, zgrid = 1;  // persistent y-pass / z-pass CTAs
    // y forward + z + y inverse pipelined through L2 in one kernel (yzy.cuh); CM_YZY
    static constexpr bool YZY = std::is_same<R, float>::value && YzyGeo<N>::OK;
    bool use_yzy = false;
    int yzy_grid = 0;
    int4* yzy_items_d = nullptr;
    int* yzy_ctr = nullptr;
    // fused K1 (k1f.cuh): x C2R + stencil + x R2C in one cluster kernel; opt-in CM_K1F=1
    static constexpr bool K1F = std::is_same<R, float>::value && K1Geo<N>::OK;
    bool use_k1f = false;
    int k1f_grid_ = 0;
    // TMA-fed persistent y pass (ypass_tma.cuh): fp32, N in {256, 512}; CM_YT=0 -> ypass
    static constexpr bool YT = std::is_same<R, float>::value && YtGeo<N>::OK;
    bool use_yt = false;
    int yt_grid = 0;
    CUtensorMap tmy_S{};
    // programmatic dependent launch between the per-iteration kernels (each
    // waits on griddepcontrol before touching its predecessor's output); opt-in:
    // measured neutral (dependents cannot start work before the predecessor
    // completes) or slower with an early trigger (waiting CTAs hold SM slots)
    bool use_pdl = std::getenv("CM_PDL") != nullptr;
    // z pass L2 prefetch lookahead (tiles) for S rows and the W / Yh blocks
    // (profiles/r2_ab_zpf.txt, 512^3: the CTA's own W / Yh block requested at
    // CTA start, 0.434 -> 0.413 ms; S rows of later tiles or W / Yh of a later
    // tile are slower; CM_Z_PFW=-1 disables)
    int z_pf = std::getenv("CM_Z_PF") ? std::atoi(std::getenv("CM_Z_PF")) : 0;
    CUtensorMap* tmz_S_d = nullptr;  // S z-box map in device memory (CM_Z_PF with CM_Z_PFT=1)
    int z_pfw = std::getenv("CM_Z_PFW") ? std::atoi(std::getenv("CM_Z_PFW")) : 0;
    cudaGraphExec_t gexec = nullptr;  // instantiated 6-iteration chunk (reused while gkey holds)
    std::vector<uint64_t> gkey;
    // fused y/x plane pairs (xyfused.cuh): fp32 power-of-two sides 256..1024
    static constexpr bool FUSE = std::is_same<R, float>::value && (N == 256 || N == 512);
    bool use_fused = false;
    int fused_grid = 0, fused_lag = 0;
    int* fcnt = nullptr;       // [2][N] per-plane producer counters
    CUtensorMap tm_spec{};     // S as [N*N rows][N/2] 8-byte elements (y column tiles)
    C* S = nullptr;
    R* W = nullptr;
    R* Wn = nullptr;
    C* Yh = nullptr;
    C* Yn = nullptr;
    C* Q0 = nullptr;           // [N][N][3] column-0 inputs, row-major
    C* Z0 = nullptr;           // forward-transformed packed column 0 [N][N]
    C* twN = nullptr;
    float4* twF4 = nullptr;    // packed {w, i w} forward / inverse tables (fp32)
    float4* twI4 = nullptr;
    double* stage = nullptr;   // fp64 staging (3L doubles)
    double* part1 = nullptr;
    double* part3 = nullptr;
    double* part_acc = nullptr;
    unsigned long long* maxes = nullptr;
    DevState* st = nullptr;
    double* trace_d = nullptr;
    int trace_rows_cap = 0;
    double* theta_d = nullptr;
    int theta_cap = 0;
    int* flags_h = nullptr;
    long long alloc_bytes = 0;

    template <typename T>
    int dalloc(T** p, size_t count) {
        const size_t b = sizeof(T) * std::max<size_t>(count, 1);
        CK(cudaMalloc((void**)p, b));
        alloc_bytes += (long long)b;
        return CM_OK;
    }

    ~Impl() override {
        if (gexec) cudaGraphExecDestroy(gexec);
        void* ps[] = {X[0], X[1], X[2], XF[0], XF[1], YF[0], YF[1], x0keep, anchor, winit, wtvf, gbuf, S, W,
                      Wn, Yh, Yn, Z0, twN, twF4, twI4, stage, part1, part3, part_acc, maxes, st, trace_d,
                      theta_d, Q0, fcnt, yzy_items_d, yzy_ctr, tmz_S_d};
        for (void* p : ps)
            if (p) cudaFree(p);
        if (flags_h) cudaFreeHost(flags_h);
        if (stream) cudaStreamDestroy(stream);
    }

    long long bytes() const override { return alloc_bytes; }

    int make_map_box(R* ptr, CUtensorMap* out, cuuint32_t bw, cuuint32_t bj, cuuint32_t bk) {
        {
            EncodeTiledFn enc = encode_tiled_fn();
            if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
            const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N};
            const cuuint64_t strides[2] = {(cuuint64_t)N * sizeof(R), (cuuint64_t)N * N * sizeof(R)};
            const cuuint32_t box[3] = {bw, bj, bk};
            const cuuint32_t es[3] = {1, 1, 1};
            CUresult r = enc(out, sizeof(R) == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                             3, ptr, dims, strides, box, es,
                             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(CM_ERR_CUDA, "tensor map encode failed");
            return CM_OK;
        }
    }
    int make_maps2(int which, R* ptr) {  // which: 0..2 X, 3..4 YF
        if constexpr (!S2) {
            return CM_OK;
        } else {
            using SG = S2GeoT<R, N>;
            CKS(make_map_box(ptr, &tm2_x[which], SG::XW, SG::XR, 1));
            if (which < 3) CKS(make_map_box(ptr, &tm2_p[which], SG::XW, SG::PR, 1));
            return CM_OK;
        }
    }

    // 3D box map over a real volume, zero OOB fill. kind 0: x box {XSW, TJ+2, TK+2};
    // 1: x_prev box {XSW, TJ+1, TK+1}; 2: interior tile {CI, TJ, TK}
    int make_map_x(R* ptr, CUtensorMap* out, int kind = 0) {
        using SG = StGeo<R, N>;
        if constexpr (!SG::V4) {
            return CM_OK;
        } else {
            const cuuint32_t bw = kind == 2 ? (cuuint32_t)SG::CI : (cuuint32_t)SG::XSW;
            const cuuint32_t bj = (cuuint32_t)(SG::TJ + (kind == 0 ? 2 : (kind == 1 ? 1 : 0)));
            const cuuint32_t bk = (cuuint32_t)(SG::TK + (kind == 0 ? 2 : (kind == 1 ? 1 : 0)));
            EncodeTiledFn enc = encode_tiled_fn();
            if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
            const cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)N, (cuuint64_t)N};
            const cuuint64_t strides[2] = {(cuuint64_t)N * sizeof(R), (cuuint64_t)N * N * sizeof(R)};
            const cuuint32_t box[3] = {bw, bj, bk};
            const cuuint32_t es[3] = {1, 1, 1};
            CUresult r = enc(out, sizeof(R) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             3, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) return fail(CM_ERR_CUDA, "tensor map (x) encode failed");
            return CM_OK;
        }
    }

    int init() override {
        n = N;
        CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        for (auto& p : X) CKS(dalloc(&p, L));
        CKS(dalloc(&x0keep, L));
        CKS(dalloc(&anchor, L));
        CKS(dalloc(&S, H));
        CKS(dalloc(&W, H));
        CKS(dalloc(&Wn, NN));
        CKS(dalloc(&Yh, H));
        CKS(dalloc(&Yn, NN));
        CKS(dalloc(&Q0, 3 * NN));
        CKS(dalloc(&Z0, NN));
        CKS(dalloc(&twN, N));
        CKS(dalloc(&stage, 3 * L));
        {
            using SG = StGeo<R, N>;
            CK(cudaFuncSetAttribute(stencil_kernel<R, N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)SG::SMEM));
            int occ = 0, dev = 0, sms = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil_kernel<R, N>, SG::NT,
                                                             SG::SMEM));
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            sweep_grid = std::max(1, std::min(SG::NTILES, sms * std::max(occ, 1)));
            CK(cudaFuncSetAttribute(xfft_kernel<R, N, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)XGeo<R, N>::SMEM));
            CK(cudaFuncSetAttribute(xfft_kernel<R, N, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)XGeo<R, N>::SMEM));
            int occx = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occx, xfft_kernel<R, N, 0>,
                                                             XGeo<R, N>::NT, XGeo<R, N>::SMEM));
            xfft_grid = sms * std::max(occx, 1);
            int occy = 0, occz = 0;
            CK(cudaFuncSetAttribute(ypass_kernel<R, N, false>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<R, N>::bytes));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occy, ypass_kernel<R, N, false>,
                                                             G::TWY * G::TY, YSmem<R, N>::bytes));
            CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FULL>,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)ZGeo<R, N>::SMEM_MAIN));
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occz, zmain_kernel<R, N, ZM_FULL>,
                                                             ZGeo<R, N>::NT, ZGeo<R, N>::SMEM_MAIN));
            ygrid = sms * std::max(occy, 1);
            zgrid = sms * std::max(occz, 1);

            if constexpr (FUSE) {
                using F = FGeo<N>;
                // opt-in: measured no faster than the separate passes at 512^3 (the
                // passes are latency/issue bound, not DRAM bound)
                use_fused = std::getenv("CM_FUSED") != nullptr;
                CK(cudaFuncSetAttribute(fused_pair_kernel<N, 0>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM));
                CK(cudaFuncSetAttribute(fused_pair_kernel<N, 1>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM));
                int occf0 = 0, occf1 = 0;
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf0, fused_pair_kernel<N, 0>, F::NT,
                                                                 F::SMEM));
                CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf1, fused_pair_kernel<N, 1>, F::NT,
                                                                 F::SMEM));
                // every CTA must be resident (consumers spin on producers); the lag
                // keeps an item's producers more than one grid ahead of it (the
                // prefetch of the next item must never wait on the current one)
                fused_grid = sms * std::max(1, std::min(occf0, occf1));
                fused_lag = std::min(N, (5 * fused_grid + 2 * F::PER_PLANE - 1) / (2 * F::PER_PLANE) + 1);
                if ((long long)(fused_lag - 1) * F::PER_PLANE < fused_grid) use_fused = false;
                CKS(dalloc(&fcnt, (size_t)2 * N));
                EncodeTiledFn enc = encode_tiled_fn();
                if (!enc) return fail(CM_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
                const cuuint64_t dims[2] = {(cuuint64_t)Nh, (cuuint64_t)N * N};
                const cuuint64_t strides[1] = {(cuuint64_t)Nh * 8};
                const cuuint32_t box[2] = {(cuuint32_t)F::TWY, (cuuint32_t)F::YBOX};
                const cuuint32_t es[2] = {1, 1};
                if (enc(&tm_spec, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, S, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
                    return fail(CM_ERR_CUDA, "tensor map encode failed (spectrum)");
            }
        }
        CKS(dalloc(&gbuf, L));
        CKS(dalloc(&part1, (size_t)std::max(NB1, sweep_grid) * NP1));
        for (int q = 0; q < 3; ++q) {
            CKS(make_map_x(X[q], &tm_x[q], 0));
            CKS(make_map_x(X[q], &tm_p[q], 1));
        }
        CKS(make_map_x(gbuf, &tm_gt, 2));
        CKS(make_map_x(anchor, &tm_at, 2));
        if constexpr (S2) {
            using SG = S2GeoT<R, N>;
            for (int q = 0; q < 3; ++q) CKS(make_maps2(q, X[q]));
            CKS(make_map_box(gbuf, &tm2_g, SG::CI, SG::TJ, 1));
            CKS(make_map_box(anchor, &tm2_a, SG::CI, SG::TJ, 1));
            CK((stencil2_prepare<N, R>()));
            int occ2 = 0, dev2 = 0, sms2 = 0;
            CK((stencil2_occupancy<N, R>(&occ2)));
            CK(cudaGetDevice(&dev2));
            CK(cudaDeviceGetAttribute(&sms2, cudaDevAttrMultiProcessorCount, dev2));
            s2_grid = std::max(1, std::min(SG::NTILES, sms2 * std::max(occ2, 1)));
        }
        CKS(dalloc(&part3, (size_t)NB3 * NP3));
        if constexpr (YZY) {
            const char* e = std::getenv("CM_YZY");
            use_yzy = e && e[0] == '1';
            CK(cudaFuncSetAttribute(yzy_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    (int)YzyGeo<N>::SMEM));
            int occ = 0, dev = 0, sms = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, yzy_kernel<N>, YzyGeo<N>::NT,
                                                             YzyGeo<N>::SMEM));
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
            yzy_grid = sms * std::max(occ, 1);
            const std::vector<int4> items = yzy_items<N>();
            CKS(dalloc(&yzy_items_d, items.size()));
            CK(cudaMemcpy(yzy_items_d, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
            CKS(dalloc(&yzy_ctr, YzyGeo<N>::NCTR));
        }
        if constexpr (K1F) {
            // opt-in (CM_K1F=1): measured 1.40 ms per 512^3 sweep against 0.96 ms for the
            // three separate kernels (one line per CTA-plane leaves the
            // warp-specialised transforms latency-bound)
            const char* e = std::getenv("CM_K1F");
            use_k1f = e && e[0] == '1';
            CK(k1f_prepare<N>());
            k1f_grid_ = k1f_grid<N>(stream);
            if (const char* g = std::getenv("CM_K1F_CLUSTERS"))  // experiments: fixed cluster count
                k1f_grid_ = std::max(1, std::min(std::atoi(g), K1Geo<N>::NTILES)) * K1Geo<N>::NCL;
            if (std::getenv("CM_K1F_DEBUG"))
                std::fprintf(stderr, "k1f: N=%d grid=%d CTAs (%d clusters of %d), smem=%zu\n", N, k1f_grid_,
                             k1f_grid_ / K1Geo<N>::NCL, K1Geo<N>::NCL, K1Geo<N>::SMEM);
            if (k1f_grid_ <= 0) use_k1f = false;
        }
        {
            // the persistent sweeps write one partial-sum slot per CTA: part1 must
            // hold the largest of their grids (the z-marching sweep's grid is known
            // only now; at 160^3 its 592 CTAs overran the 400 slots allocated above)
            const int need = std::max(std::max(NB1, sweep_grid), std::max(s2_grid, k1f_grid_));
            if (need > std::max(NB1, sweep_grid)) {
                CK(cudaFree(part1));
                part1 = nullptr;
                CKS(dalloc(&part1, (size_t)need * NP1));
            }
        }
        if constexpr (YT) {
            using YG_ = YtGeo<N>;
            const char* e = std::getenv("CM_YT");
            use_yt = !(e && e[0] == '0');
            CK(yt_prepare<N>());
            int occt = 0, devt = 0, smst = 0;
            CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occt, ytma_kernel<N, true>, YG_::NT,
                                                             YG_::SMEM));
            CK(cudaGetDevice(&devt));
            CK(cudaDeviceGetAttribute(&smst, cudaDevAttrMultiProcessorCount, devt));
            yt_grid = std::max(1, std::min(YG_::NTILES, smst * std::max(occt, 1)));
            CKS(yt_make_map(S, N, YG_::TW, YG_::BOXB, &tmy_S));
            if (z_pf > 0 && std::getenv("CM_Z_PFT")) {
                CUtensorMap m{};
                CKS(yt_make_map(S, N, ZGeo<R, N>::TW, 1, &m, N < 256 ? N : 256));
                CKS(dalloc(reinterpret_cast<char**>(&tmz_S_d), sizeof(CUtensorMap)));
                CK(cudaMemcpy(tmz_S_d, &m, sizeof(m), cudaMemcpyHostToDevice));
            }
        }
        CKS(dalloc(&part_acc, 2 * 148 * 32));
        CKS(dalloc(&maxes, 4));
        CKS(dalloc(&st, 1));
        CK(cudaHostAlloc((void**)&flags_h, sizeof(int) * LOOK, cudaHostAllocDefault));
        for (auto& p : X) CK(cudaMemsetAsync(p, 0, sizeof(R) * L, stream));
        // twiddles exp(-2 pi i q / N) computed in fp64 on the host, rounded once
        std::vector<C> tw(N);
        for (int q = 0; q < N; ++q) {
            const double a = -2.0 * M_PI * (double)q / (double)N;
            tw[q].x = R(std::cos(a));
            tw[q].y = R(std::sin(a));
        }
        CK(cudaMemcpyAsync(twN, tw.data(), sizeof(C) * N, cudaMemcpyHostToDevice, stream));
        if constexpr (sizeof(R) == 4) {
            std::vector<float4> f(N), iv(N);
            for (int q = 0; q < N; ++q) {
                const double a = -2.0 * M_PI * (double)q / (double)N;
                const float c = (float)std::cos(a), sn = (float)std::sin(a);
                f[q] = make_float4(c, sn, -sn, c);     // w, i w
                iv[q] = make_float4(c, -sn, sn, c);    // conj w, i conj w
            }
            CKS(dalloc(&twF4, N));
            CKS(dalloc(&twI4, N));
            CK(cudaMemcpy(twF4, f.data(), sizeof(float4) * N, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(twI4, iv.data(), sizeof(float4) * N, cudaMemcpyHostToDevice));
        }
        CK(cudaFuncSetAttribute(ypass_kernel<R, N, true>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<R, N>::bytes));
        CK(cudaFuncSetAttribute(ypass_kernel<R, N, false>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)YSmem<R, N>::bytes));
        using ZG = ZGeo<R, N>;
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FULL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FIT>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        CK(cudaFuncSetAttribute(zmain_kernel<R, N, ZM_FWD>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_MAIN));
        CK(cudaFuncSetAttribute(zcol0_kernel<R, N, ZM_FULL>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_COL0));
        CK(cudaFuncSetAttribute(zcol0_kernel<R, N, ZM_FIT>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ZG::SMEM_COL0));
        CK(cudaStreamSynchronize(stream));
        return CM_OK;
    }

    // ---- launch helpers ----------------------------------------------------------
    XParams<R> xp() const {
        XParams<R> p{};
        p.S = S;
        p.twN = twN;
        p.invL = 1.0 / (double)L;
        return p;
    }
    template <int MODE>
    int launch_x(const XParams<R>& p) {
        xline_kernel<R, N, MODE><<<NB1, G::LPC * G::TX, 0, stream>>>(p);
        CK(cudaGetLastError());
        return CM_OK;
    }
    int launch_y(bool fwd, DevState* s) {
        if constexpr (YT) {
            if (use_yt) {
                const int* stop = s ? (fwd ? &s->done_y : &s->done) : nullptr;
                if (fwd)
                    CK(launch_pdl(use_pdl, ytma_kernel<N, true>, dim3(yt_grid), dim3(YtGeo<N>::NT),
                                  YtGeo<N>::SMEM, stream, S, twN, stop, tmy_S));
                else
                    CK(launch_pdl(use_pdl, ytma_kernel<N, false>, dim3(yt_grid), dim3(YtGeo<N>::NT),
                                  YtGeo<N>::SMEM, stream, S, twN, stop, tmy_S));
                return CM_OK;
            }
        }
        const SpecLayout nat = spec_layout((long long)N * Nh, 0, N, Nh);
        YParams<R> p{S, twN, fwd ? twF4 : twI4, s ? (fwd ? &s->done_y : &s->done) : nullptr,
                     nullptr, nat, nat, N, 0, Nh / G::TWY};
        const int grid = std::min((Nh / G::TWY) * N, ygrid);  // persistent
        if (fwd)
            CK(launch_pdl(use_pdl, ypass_kernel<R, N, true>, dim3(grid), dim3(G::TWY * G::TY),
                          YSmem<R, N>::bytes, stream, p));
        else
            CK(launch_pdl(use_pdl, ypass_kernel<R, N, false>, dim3(grid), dim3(G::TWY * G::TY),
                          YSmem<R, N>::bytes, stream, p));
        return CM_OK;
    }
    // x-line transforms: dir 0 C2R (S -> g * invL), dir 1 R2C (real -> S)
    int launch_xfft(int dir, R* real, const int* stop) {
        using XG = XGeo<R, N>;
        XfParams<R> p{S, real, twN, dir == 0 ? twI4 : twF4, stop, 1.0 / (double)L, N * N};
        const int grid = std::min(XG::NB, xfft_grid);
        if (dir == 0)
            CK(launch_pdl(use_pdl, xfft_kernel<R, N, 0>, dim3(grid), dim3(XG::NT), XG::SMEM, stream, p));
        else
            CK(launch_pdl(use_pdl, xfft_kernel<R, N, 1>, dim3(grid), dim3(XG::NT), XG::SMEM, stream, p));
        return CM_OK;
    }

    // fused plane pairs: dir 0 = y inverse + x C2R (S -> g), dir 1 = x R2C + y forward
    int launch_fused(int dir, R* real, const int* stop) {
        if constexpr (FUSE) {
            using F = FGeo<N>;
            CK(cudaMemsetAsync(fcnt + (size_t)dir * N, 0, sizeof(int) * N, stream));
            FusedParams fp{reinterpret_cast<float2*>(S), reinterpret_cast<float*>(real),
                           reinterpret_cast<const float2*>(twN), stop, fcnt + (size_t)dir * N,
                           (float)(1.0 / (double)L), fused_lag};
            if (dir == 0)
                fused_pair_kernel<N, 0><<<fused_grid, F::NT, F::SMEM, stream>>>(fp, tm_spec);
            else
                fused_pair_kernel<N, 1><<<fused_grid, F::NT, F::SMEM, stream>>>(fp, tm_spec);
            CK(cudaGetLastError());
            return CM_OK;
        } else {
            (void)dir; (void)real; (void)stop;
            return fail(CM_ERR_UNSUPPORTED, "fused plane pairs: fp32 N in {256, 512} only");
        }
    }

    // K3: z pass (main tiles, then the packed column 0 with its Friedel mates)
    template <int MODE>
    int launch_z(double* part, DevState* s) {
        using ZG = ZGeo<R, N>;
        ZMParams<R> p{S, Z0, W, Wn, Yh, Yn, twN, twF4, twI4, part, s, N, Q0, Nh, 0};
        p.pf = z_pf;
        p.pfw = z_pfw;
        p.tmS = tmz_S_d;
        dim3 grid(Nh / ZG::TW, N);
        CK(launch_pdl(use_pdl, zmain_kernel<R, N, MODE>, grid, dim3(ZG::NT), ZG::SMEM_MAIN, stream, p));
        if constexpr (MODE != ZM_FWD)
            CK(launch_pdl(use_pdl, zcol0_kernel<R, N, MODE>, dim3(N / 2 + 1), dim3(ZG::NT0),
                          ZG::SMEM_COL0, stream, p));
        return CM_OK;
    }
    // y forward (of the spectrum in S) + z pass + y inverse, one launch (yzy.cuh)
    int launch_yzy(double* part, DevState* s) {
        if constexpr (YZY) {
            ZMParams<R> p{S, Z0, W, Wn, Yh, Yn, twN, twF4, twI4, part, s, N, Q0, Nh, 0};
            CK(cudaMemsetAsync(yzy_ctr, 0, sizeof(int) * YzyGeo<N>::NCTR, stream));
            yzy_kernel<N><<<yzy_grid, YzyGeo<N>::NT, YzyGeo<N>::SMEM, stream>>>(p, yzy_items_d, yzy_ctr);
            CK(cudaGetLastError());
        }
        return CM_OK;
    }
    int upload_real(const double* host, R* dst) {
        CKS(xfer.h2d(stage, host, sizeof(double) * L, stream));
        to_real_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(stage, dst, L);
        CK(cudaGetLastError());
        return CM_OK;
    }
    int download_real(const R* src, double* host) {
        to_double_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(src, stage, L);
        CK(cudaGetLastError());
        CKS(xfer.d2h(host, stage, sizeof(double) * L, stream));
        return CM_OK;
    }

    // ---- accumulator ---------------------------------------------------------------
    int set_accumulator(const double* w, const double* y, int finalized) override {
        CKS(xfer.h2d(stage, w, sizeof(double) * L, stream));
        CKS(xfer.h2d(stage + L, y, sizeof(double) * 2 * L, stream));
        return commit_acc_stage(finalized);
    }
    double* acc_stage() override { return stage; }
    // the accumulator in `stage` (weight [L], numerator [L] complex interleaved),
    // written there by set_accumulator's upload or by the device backprojection
    int commit_acc_stage(int finalized) override {
        CK(cudaMemsetAsync(maxes, 0, sizeof(unsigned long long) * 4, stream));
        const int blocks = grid_for(NN * (Nh + 1), 256);
        convert_acc_kernel<R><<<blocks, 256, 0, stream>>>(N, stage, stage + L, W, Wn, Yh, Yn,
                                                          part_acc, maxes, Q0, ZGeo<R, N>::TW);
        CK(cudaGetLastError());
        std::vector<double> parts(2 * (size_t)blocks);
        unsigned long long mx[4];
        CK(cudaMemcpyAsync(parts.data(), part_acc, sizeof(double) * parts.size(),
                           cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(mx, maxes, sizeof(mx), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double sw = 0.0, sz = 0.0;
        for (int b = 0; b < blocks; ++b) {
            sw += parts[2 * b];
            sz += parts[2 * b + 1];
        }
        double worst, scale, wmax;
        std::memcpy(&worst, &mx[0], 8);
        std::memcpy(&scale, &mx[1], 8);
        std::memcpy(&wmax, &mx[2], 8);
        residue = scale > 0.0 ? worst / scale : 0.0;
        max_weight = wmax;
        s_n = sw / (double)L;
        s_y = std::sqrt(sz) / (double)L; // Parseval: RMS = sqrt(sum |Z_H|^2 / L) / sqrt(L)
        acc_set = true;
        acc_finalized = finalized != 0;
        return CM_OK;
    }

    int set_volumes(const double* xi, const double* xa) override {
        CKS(upload_real(xi, x0keep));
        anchor_is_init = (xa == xi);
        if (anchor_is_init) {
            CK(cudaMemcpyAsync(anchor, x0keep, sizeof(R) * L, cudaMemcpyDeviceToDevice, stream));
        } else {
            CKS(upload_real(xa, anchor));
        }
        CK(cudaStreamSynchronize(stream));
        vol_set = true;
        return CM_OK;
    }

    int require_acc() {
        if (!acc_set) return fail(CM_ERR_STATE, "accumulator not set");
        if (!acc_finalized || residue > 1e-9)
            return fail(CM_ERR_NON_HERMITIAN, "accumulator is not Friedel-finalized");
        return CM_OK;
    }

    // ---- the solver ------------------------------------------------------------------
    int solve(const cm_reg_config* c, cm_trace_row* trace, int cap, cm_solve_stats* stats) override {
        NvtxRange nvtx_solve("cm_m_step_solve");
        CKS(validate(c));
        CKS(require_acc());
        if (!vol_set) return fail(CM_ERR_STATE, "volumes not set");
        const int K = c->inner_iters;
        const bool lipschitz = c->step_rule == 0;
        const bool fista = c->momentum >= 1;
        const bool convex = c->convex_mode != 0;
        const bool want_trace = trace != nullptr && cap > 0;
        const bool audit = !fista && (lipschitz || want_trace || c->tol_kind == 1);
        const bool refresh_inner = (c->refresh == 0) && !convex;
        // max w_tv is attained at voxel (0,0,0), where Dx = 0 under the
        // replicate rule, so max w_tv = 1/eps' exactly (1 in convex mode)
        const double max_wtv = convex ? 1.0 : 1.0 / c->eps_prime;
        const double lr = lipschitz ? 1.0 / (2.0 * max_weight + 2.0 * c->gamma +
                                             12.0 * c->beta * max_wtv / c->mu)
                                    : c->fixed_step;
        double slack = c->audit_slack;
        if (!(slack > 0.0)) slack = sizeof(R) == 8 ? 1e-9 : 1e-6;

        if (fista) {
            for (auto& p : XF)
                if (!p) CKS(dalloc(&p, L));
            for (int q = 0; q < 2; ++q)
                if (!YF[q]) {
                    CKS(dalloc(&YF[q], L));
                    CKS(make_map_x(YF[q], &tm_x[3 + q]));
                    CKS(make_maps2(3 + q, YF[q]));
                }
        }
        const bool need_winit = (c->refresh == 1) && !convex && !anchor_is_init;
        if (need_winit && !winit) CKS(dalloc(&winit, L));
        if (want_trace && trace_rows_cap < K) {
            if (trace_d) cudaFree(trace_d);
            trace_d = nullptr;
            CKS(dalloc(&trace_d, (size_t)K * 15));
            trace_rows_cap = K;
        }
        if (fista && theta_cap < K + 1) {
            if (theta_d) cudaFree(theta_d);
            theta_d = nullptr;
            CKS(dalloc(&theta_d, (size_t)K + 1));
            theta_cap = K + 1;
        }
        if (fista) {
            std::vector<double> th(K + 1);
            double tk = 1.0;
            for (int q = 0; q <= K; ++q) {
                const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tk * tk));
                th[q] = (tk - 1.0) / tn;
                tk = tn;
            }
            CK(cudaMemcpyAsync(theta_d, th.data(), sizeof(double) * (K + 1),
                               cudaMemcpyHostToDevice, stream));
        }

        // starting point and weight source
        R* const x0buf = fista ? XF[0] : X[0];
        CK(cudaMemcpyAsync(x0buf, x0keep, sizeof(R) * L, cudaMemcpyDeviceToDevice, stream));
        if (fista)
            CK(cudaMemcpyAsync(YF[0], x0keep, sizeof(R) * L, cudaMemcpyDeviceToDevice, stream));
        if (need_winit)
            CK(cudaMemcpyAsync(winit, x0keep, sizeof(R) * L, cudaMemcpyDeviceToDevice, stream));
        const R* wfixed = (c->refresh == 1 && !convex) ? (anchor_is_init ? anchor : winit) : nullptr;
        if (wfixed) {
            // frozen weights (Refresh::per_m_step, regularizer.cpp:178-179): the
            // w_tv field of x_init once per solve; w_l1 comes from x_init itself
            if (!wtvf) CKS(dalloc(&wtvf, L));
            XParams<R> wp = xp();
            wp.xcur = wfixed;
            wp.wsrc = wfixed;
            wp.eps = c->eps;
            wp.eps_prime = c->eps_prime;
            wp.xnext = fista ? YF[1] : X[2];  // w_l1 scratch, overwritten by the solve
            wp.ynext = wtvf;
            CKS(launch_x<XM_WEIGHTS>(wp));
        }

        DevState hs{};
        hs.iter = 0;
        hs.max_iters = K;
        hs.diverged_iter = -1;
        hs.audit = audit;
        hs.check_diverge = audit && lipschitz;
        hs.tol_kind = c->tol_kind;
        if (fista && hs.tol_kind == 1) hs.tol_kind = 2; // no surrogate audit under momentum
        hs.fista = fista;
        hs.restart = c->momentum == 2;
        hs.mom_base = 0;
        hs.restarts = 0;
        hs.refresh_inner = refresh_inner;
        hs.tol = c->tol;
        hs.audit_slack = slack;
        hs.step = lr;
        CK(cudaMemcpyAsync(st, &hs, sizeof(hs), cudaMemcpyHostToDevice, stream));

        const bool need_part1 = audit || hs.tol_kind == 2 || hs.restart;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, stream));
        int launches = 0;

        // spectrum of the starting point: x R2C, y forward (yzy: + z and y inverse
        // of iteration 0)
        const bool yzy = YZY && use_yzy && !use_fused && !profiling;
        if (yzy) {
            CKS(launch_xfft(1, fista ? YF[0] : X[0], nullptr));
            CKS(launch_yzy(audit ? part3 : nullptr, st));
            launches += 2;
        } else if (use_fused) {
            CKS(launch_fused(1, fista ? YF[0] : X[0], nullptr));
            launches += 1;
        } else {
            CKS(launch_xfft(1, fista ? YF[0] : X[0], nullptr));
            CKS(launch_y(true, nullptr));
            launches += 2;
        }

        cudaEvent_t pev[8] = {};
        if (profiling)
            for (auto& e : pev) CK(cudaEventCreate(&e));
        static const char* const kPhase[8] = {"z_pass", "y_inverse", "x_c2r", "stencil",
                                              "finalize", "x_r2c", "y_forward", "end"};
        auto mark = [&](int q) -> int {
            if (profiling) {
                CK(cudaEventRecord(pev[q], stream));
                // per-kernel NVTX ranges in the profiling solve (kernels launched one by one)
                if (q > 0) nvtxRangePop();
                if (q < 7) nvtxRangePushA(kPhase[q]);
            }
            return CM_OK;
        };
        auto sweep_and_finalize = [&](int g, cudaEvent_t mid) -> int {
            (void)mid;
            // K1a: x-line C2R -> data gradient (real space, / L); fused: the y
            // inverse of the same planes ran in the same kernel (mark 2 -> 3 is empty)
            const bool k1f = K1F && use_k1f && !use_fused;
            if (!use_fused && !k1f) CKS(launch_xfft(0, gbuf, &st->done));
            CKS(mark(3));
            // K1b: stencil sweep
            StencilParams<R> p{};
            p.g = gbuf;
            p.st = st;
            p.lr = lr;
            p.alpha = c->alpha;
            p.beta = c->beta;
            p.gamma = c->gamma;
            p.eps = c->eps;
            p.eps_prime = c->eps_prime;
            p.mu = c->mu;
            p.convex = convex;
            p.audit = audit;
            p.fista = fista;
            p.trace_full = want_trace;
            p.steptol = hs.tol_kind == 2;
            p.koff = 0;
            p.nk = N;
            p.zshift = 0;
            p.anchor = anchor;
            p.part = need_part1 ? part1 : nullptr;
            const CUtensorMap* tmx = nullptr;
            const CUtensorMap* tmp = nullptr;
            R* spec_src = nullptr;
            if (fista) {
                p.xcur = YF[g % 2];
                p.xold = XF[g % 2];
                p.xnext = XF[(g + 1) % 2];
                p.ynext = YF[(g + 1) % 2];
                p.theta = theta_d;
                tmx = &tm_x[3 + g % 2];
                tmp = tmx;
                spec_src = YF[(g + 1) % 2];
            } else {
                p.xcur = X[g % 3];
                p.xnext = X[(g + 1) % 3];
                p.xprev = (audit && refresh_inner) ? X[(g + 2) % 3] : nullptr;
                tmx = &tm_x[g % 3];
                tmp = &tm_p[(g + 2) % 3];
                spec_src = X[(g + 1) % 3];
            }
            if (wfixed) {
                p.wtvf = wtvf;
                p.wl1src = wfixed;
            }
            const bool use_s2 = S2 && std::getenv("CM_STENCIL1") == nullptr;
            if constexpr (K1F) {
                if (k1f) {
                    const int xi = fista ? 3 + g % 2 : g % 3;
                    const int pi = fista ? 0 : (g + 2) % 3;
                    CK(k1f_launch<N>(p, reinterpret_cast<float2*>(S), reinterpret_cast<const float2*>(twN),
                                     k1f_grid_, stream, tm2_x[xi], tm2_p[pi], tm2_a));
                }
            }
            if constexpr (S2) {
                if (use_s2 && !k1f) {
                    const int xi = fista ? 3 + g % 2 : g % 3;
                    const int pi = fista ? 0 : (g + 2) % 3;
                    CK(stencil2_launch<N>(p, s2_grid, stream, tm2_x[xi], tm2_p[pi], tm2_g, tm2_a,
                                          use_pdl));
                }
            }
            if (!use_s2 && !k1f)
                stencil_kernel<R, N><<<sweep_grid, StGeo<R, N>::NT, StGeo<R, N>::SMEM, stream>>>(
                    p, *tmx, *tmp, tm_gt, tm_at);
            CK(cudaGetLastError());
            CKS(mark(4));
            // FIN
            FinParams f{};
            f.st = st;
            f.part1 = need_part1 ? part1 : nullptr;
            f.nb1 = k1f ? k1f_grid_ : use_s2 ? s2_grid : sweep_grid;  // partial slots of the sweep
            f.part3 = audit ? part3 : nullptr;
            f.nb3 = NB3;
            f.trace = want_trace ? trace_d : nullptr;
            f.alpha = c->alpha;
            f.beta = c->beta;
            f.gamma = c->gamma;
            f.invL = 1.0 / (double)L;
            f.epilogue = 0;
            CK(launch_pdl(use_pdl, finalize_kernel, dim3(1), dim3(FIN_THREADS), 0, stream, f));
            CKS(mark(5));
            // K1c: x-line R2C of the new iterate (FISTA: of y_{k+1}); fused: + y forward
            if (use_fused) CKS(launch_fused(1, spec_src, &st->done_y));
            else if (!k1f) CKS(launch_xfft(1, spec_src, &st->done_y));  // k1f: done in the sweep
            CKS(mark(6));
            return CM_OK;
        };
        auto iteration = [&](int g) -> int {
            if (yzy) {  // z + y inverse ran in the previous yzy launch
                CKS(sweep_and_finalize(g, nullptr));                // K1 + FIN
                CKS(launch_yzy(audit ? part3 : nullptr, st));      // K2 + next K3 + K4
                return CM_OK;
            }
            CKS(launch_z<ZM_FULL>(audit ? part3 : nullptr, st));  // K3
            if (use_fused) CKS(launch_fused(0, gbuf, &st->done));  // K4 + K1a
            else CKS(launch_y(false, st));                         // K4
            CKS(sweep_and_finalize(g, nullptr));                   // K1 + FIN
            if (!use_fused) CKS(launch_y(true, st));               // K2
            return CM_OK;
        };

        const int per_iter = yzy ? (K1F && use_k1f ? 3 : 5)
                                 : (use_fused || (K1F && use_k1f)) ? 6 : 8;  // kernels per iteration
        const bool use_graph = std::getenv("CM_NO_GRAPH") == nullptr && !profiling;
        const int chunk = 6;
        const int nchunks = (K + chunk - 1) / chunk;
        if (profiling) {
            // per-kernel timing: same kernels, launched one by one between events
            for (int q = 0; q < 8; ++q) prof_ms[q] = 0.0;
            prof_iters = 0;
            for (int g = 0; g < K; ++g) {
                CKS(mark(0));
                CKS(launch_z<ZM_FULL>(audit ? part3 : nullptr, st));
                CKS(mark(1));
                if (use_fused) CKS(launch_fused(0, gbuf, &st->done));
                else CKS(launch_y(false, st));
                CKS(mark(2));
                CKS(sweep_and_finalize(g, nullptr));
                if (!use_fused) CKS(launch_y(true, st));
                CKS(mark(7));
                CK(cudaEventSynchronize(pev[7]));
                for (int q = 0; q < 7; ++q) {
                    float m = 0.f;
                    CK(cudaEventElapsedTime(&m, pev[q], pev[q + 1]));
                    prof_ms[q] += m;
                }
                ++prof_iters;
                launches += per_iter;
            }
            for (auto& e : pev) cudaEventDestroy(e);
        } else if (use_graph) {
            // the captured chunk depends only on the values baked into its kernel
            // parameters: reuse the instantiated graph while they are unchanged
            std::vector<uint64_t> key;
            auto put = [&](double v) {
                uint64_t u;
                std::memcpy(&u, &v, 8);
                key.push_back(u);
            };
            for (double v : {c->alpha, c->beta, c->gamma, c->eps, c->eps_prime, c->mu, c->fixed_step,
                             lr, slack})
                put(v);
            for (long long v : {(long long)c->step_rule, (long long)c->refresh, (long long)c->convex_mode,
                                (long long)c->momentum, (long long)hs.tol_kind, (long long)want_trace,
                                (long long)audit, (long long)use_fused, (long long)use_pdl,
                                (long long)(std::getenv("CM_STENCIL1") != nullptr),
                                (long long)(uintptr_t)trace_d, (long long)(uintptr_t)theta_d,
                                (long long)(uintptr_t)wfixed})
                key.push_back((uint64_t)v);
            if (!(gexec && key == gkey)) {
                if (gexec) cudaGraphExecDestroy(gexec);
                gexec = nullptr;
                cudaGraph_t graph;
                CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
                int rc = CM_OK;
                for (int g = 0; g < chunk && rc == CM_OK; ++g) rc = iteration(g);
                cudaError_t ce = cudaStreamEndCapture(stream, &graph);
                if (rc != CM_OK) return rc;
                CK(ce);
                const cudaError_t ie = cudaGraphInstantiate(&gexec, graph, 0);
                cudaGraphDestroy(graph);
                CK(ie);
                gkey = key;
            }
            cudaGraphExec_t exec = gexec;
            std::vector<cudaEvent_t> ev(LOOK);
            for (auto& e : ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            for (int q = 0; q < nchunks; ++q) {
                if (q >= LOOK) {
                    CK(cudaEventSynchronize(ev[q % LOOK]));
                    if (flags_h[q % LOOK]) break;
                }
                CK(cudaGraphLaunch(exec, stream));
                launches += per_iter * chunk;
                CK(cudaMemcpyAsync(&flags_h[q % LOOK], &st->done, sizeof(int),
                                   cudaMemcpyDeviceToHost, stream));
                CK(cudaEventRecord(ev[q % LOOK], stream));
            }
            CK(cudaStreamSynchronize(stream));
            for (auto& e : ev) cudaEventDestroy(e);
        } else {
            for (int g = 0; g < K; ++g) {
                CKS(iteration(g % 6));
                launches += per_iter;
            }
        }

        DevState rs;
        CK(cudaMemcpyAsync(&rs, st, sizeof(rs), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        if (audit && rs.stop_reason == 1) {
            // close the last trace row: fit(x_K) and the penalties of x_K under the
            // weights of iteration K-1 (regularizer.cpp:208)
            CKS(launch_z<ZM_FIT>(part3, nullptr));
            // the penalties: the z-marching sweep in its objective-only mode (the
            // same partial slots as a per-iteration audit; 1.9 -> ~0.4 ms at 512^3
            // against the scalar xline epilogue), else the generic line kernel
            int nb1 = NB1;
            bool done_s2 = false;
            if constexpr (S2) {
                if (!fista && std::getenv("CM_STENCIL1") == nullptr && std::getenv("CM_EPI_XLINE") == nullptr) {
                    StencilParams<R> q{};
                    q.g = gbuf;  // read by the ring, unused without an update
                    q.st = nullptr;
                    q.lr = lr;
                    q.alpha = c->alpha;
                    q.beta = c->beta;
                    q.gamma = c->gamma;
                    q.eps = c->eps;
                    q.eps_prime = c->eps_prime;
                    q.mu = c->mu;
                    q.convex = convex;
                    q.audit = 1;
                    q.trace_full = want_trace;
                    q.anchor = anchor;
                    q.part = part1;
                    q.koff = 0;
                    q.nk = N;
                    q.zshift = 0;
                    q.obj_only = 1;
                    q.xcur = X[K % 3];
                    q.xnext = X[(K + 1) % 3];
                    q.xprev = refresh_inner ? X[(K + 2) % 3] : nullptr;
                    if (wfixed) {
                        q.wtvf = wtvf;
                        q.wl1src = wfixed;
                    }
                    CK(stencil2_launch<N>(q, s2_grid, stream, tm2_x[K % 3], tm2_p[(K + 2) % 3], tm2_g,
                                          tm2_a));
                    nb1 = s2_grid;
                    done_s2 = true;
                }
            }
            if (!done_s2) {
                XParams<R> p = xp();
                p.eps = c->eps;
                p.eps_prime = c->eps_prime;
                p.mu = c->mu;
                p.convex = convex;
                p.audit = 1;
                p.anchor = anchor;
                p.part = part1;
                p.xcur = X[K % 3];
                p.xprev = refresh_inner ? X[(K + 2) % 3] : nullptr;
                p.wsrc = wfixed ? wfixed : p.xcur;
                CKS(launch_x<XM_OBJ>(p));
            }
            FinParams f{};
            f.st = st;
            f.part1 = part1;
            f.nb1 = nb1;
            f.part3 = part3;
            f.nb3 = NB3;
            f.trace = want_trace ? trace_d : nullptr;
            f.alpha = c->alpha;
            f.beta = c->beta;
            f.gamma = c->gamma;
            f.invL = 1.0 / (double)L;
            f.epilogue = 1;
            finalize_kernel<<<1, FIN_THREADS, 0, stream>>>(f);
            CK(cudaGetLastError());
            launches += 3;
            CK(cudaMemcpyAsync(&rs, st, sizeof(rs), cudaMemcpyDeviceToHost, stream));
        }
        CK(cudaEventRecord(e1, stream));
        CK(cudaStreamSynchronize(stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);

        const int rows = std::min(rs.rows, want_trace ? cap : 0);
        if (want_trace && rows > 0) {
            std::vector<double> tr((size_t)rows * 15);
            CK(cudaMemcpy(tr.data(), trace_d, sizeof(double) * tr.size(), cudaMemcpyDeviceToHost));
            for (int r = 0; r < rows; ++r) {
                std::memcpy(trace[r].before, &tr[15 * r], 7 * sizeof(double));
                std::memcpy(trace[r].after, &tr[15 * r + 7], 7 * sizeof(double));
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
            stats->kernel_launches = launches;
        }
        if (rs.stop_reason == 3)
            return fail(CM_ERR_STEP_DIVERGED, "m_step: frozen-weight objective increased");
        return CM_OK;
    }

    float* mrc_landing(int which) override {
        if constexpr (sizeof(R) == 4)
            return reinterpret_cast<float*>(which == 0 ? x0keep : anchor);
        else
            return reinterpret_cast<float*>(stage);
    }
    int mrc_commit(int which) override {
        if constexpr (sizeof(R) == 8) {
            if (which < 2) {
                f32_to_real_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(
                    reinterpret_cast<const float*>(stage), which == 0 ? x0keep : anchor, L);
                CK(cudaGetLastError());
            }
        }
        if (which == 2)
            CK(cudaMemcpyAsync(anchor, x0keep, sizeof(R) * L, cudaMemcpyDeviceToDevice, stream));
        if (which != 0) {
            anchor_is_init = which == 2;
            vol_set = true;
        }
        return CM_OK;
    }
    const float* mrc_result_f32() override {
        if (!vol_set || !result_valid) return nullptr;
        const R* src = last_fista ? XF[last_iter % 2] : X[last_iter % 3];
        if constexpr (sizeof(R) == 4) {
            return reinterpret_cast<const float*>(src);
        } else {
            float* dst = reinterpret_cast<float*>(stage);
            real_to_f32_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(src, dst, L);
            return cudaGetLastError() == cudaSuccess ? dst : nullptr;
        }
    }

    int get_volume(double* out) override {
        if (!vol_set || !result_valid) return fail(CM_ERR_STATE, "no solver result resident");
        const R* src = last_fista ? XF[last_iter % 2] : X[last_iter % 3];
        return download_real(src, out);
    }

    // ---- component entry points ---------------------------------------------------------
    int spectrum_of(R* x) { // S <- x R2C, y forward (the z pass follows)
        CKS(launch_xfft(1, x, nullptr));
        CKS(launch_y(true, nullptr));
        return CM_OK;
    }

    int data_gradient(const double* x, double* out) override {
        CKS(require_acc());
        CKS(upload_real(x, X[0]));
        CKS(spectrum_of(X[0]));
        CKS(launch_z<ZM_FULL>(nullptr, nullptr));
        CKS(launch_y(false, nullptr));
        CKS(launch_xfft(0, X[1], nullptr));
        result_valid = false; // X[] reused as scratch; x0keep / anchor untouched
        return download_real(X[1], out);
    }

    int weights(const double* x, double eps, double epsp, int convex, double* wl1,
                double* wtv) override {
        result_valid = false;
        CKS(upload_real(x, X[0]));
        XParams<R> p = xp();
        p.xcur = X[0];
        p.wsrc = X[0];
        p.eps = eps;
        p.eps_prime = epsp;
        p.convex = convex;
        p.xnext = X[1];
        p.ynext = X[2];
        CKS(launch_x<XM_WEIGHTS>(p));
        CKS(download_real(X[1], wl1));
        return download_real(X[2], wtv);
    }

    int tv(const double* x, double mu, const double* wtv, double* value, double* grad) override {
        result_valid = false;
        CKS(upload_real(x, X[0]));
        if (wtv) CKS(upload_real(wtv, X[2]));
        XParams<R> p = xp();
        p.xcur = X[0];
        p.wsrc = X[0];
        p.mu = mu;
        p.eps = 1.0;
        p.eps_prime = 1.0;
        p.convex = wtv ? 0 : 1;
        p.wtvf = wtv ? X[2] : nullptr;
        if (grad) {
            p.xnext = X[1];
            CKS(launch_x<XM_TVGRAD>(p));
            CKS(download_real(X[1], grad));
        }
        if (value) {
            p.part = part1;
            CKS(launch_x<XM_OBJ>(p));
            std::vector<double> h((size_t)NB1 * NP1);
            CK(cudaMemcpyAsync(h.data(), part1, sizeof(double) * h.size(),
                               cudaMemcpyDeviceToHost, stream));
            CK(cudaStreamSynchronize(stream));
            double s = 0.0;
            for (int b = 0; b < NB1; ++b) s += h[(size_t)b * NP1 + 1];
            *value = s;
        }
        return CM_OK;
    }

    int prox(const double* x, const double* t, double* out) override {
        CK(cudaMemcpyAsync(stage, x, sizeof(double) * L, cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(stage + L, t, sizeof(double) * L, cudaMemcpyHostToDevice, stream));
        prox_kernel<<<grid_for(L, 256), 256, 0, stream>>>(stage, stage + L, stage + 2 * L, L);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, stage + 2 * L, sizeof(double) * L, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return CM_OK;
    }

    int objective(const double* x, const cm_reg_config* c, const double* anc, const double* wsrc,
                  double* out7) override {
        result_valid = false;
        CKS(validate(c));
        CKS(require_acc());
        CKS(upload_real(x, X[0]));
        CKS(upload_real(anc, X[1]));
        CKS(upload_real(wsrc, X[2]));
        CKS(spectrum_of(X[0]));
        CKS(launch_z<ZM_FIT>(part3, nullptr));
        XParams<R> p = xp();
        p.xcur = X[0];
        p.anchor = X[1];
        p.wsrc = X[2];
        p.eps = c->eps;
        p.eps_prime = c->eps_prime;
        p.mu = c->mu;
        p.convex = c->convex_mode;
        p.audit = 1;
        p.part = part1;
        CKS(launch_x<XM_OBJ>(p));
        std::vector<double> h1((size_t)NB1 * NP1), h3((size_t)NB3 * NP3);
        CK(cudaMemcpyAsync(h1.data(), part1, sizeof(double) * h1.size(), cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(h3.data(), part3, sizeof(double) * h3.size(), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        double s[NP1] = {}, q = 0.0, cr = 0.0;
        for (int b = 0; b < NB1; ++b)
            for (int k = 0; k < NP1; ++k) s[k] += h1[(size_t)b * NP1 + k];
        for (int b = 0; b < NB3; ++b) {
            q += h3[(size_t)b * NP3];
            cr += h3[(size_t)b * NP3 + 1];
        }
        out7[0] = (q - 2.0 * cr) / (double)L;
        out7[1] = c->alpha * s[0];
        out7[2] = c->beta * s[1];
        out7[3] = c->beta * s[2];
        out7[4] = c->gamma * s[5];
        out7[5] = c->alpha * s[3];
        out7[6] = c->beta * s[4];
        return CM_OK;
    }

    // full complex grid of fft3(x) (or fft3_centered) of a device volume -> host
    int spectrum_to_host(R* x, double* out, int centered) {
        CKS(spectrum_of(x));
        CKS(launch_z<ZM_FWD>(nullptr, nullptr));
        unpack_full_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(N, S, stage, centered);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, stage, sizeof(double) * 2 * L, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return CM_OK;
    }

    // fft3 / fft3_centered (fourier.cpp:59-66, 109) of a host volume; the upload
    // goes to an iterate buffer that does not hold the resident solve result
    int fft3(const double* x, double* out, int centered) override {
        R* buf = X[0];
        if (result_valid && !last_fista && X[last_iter % 3] == buf) buf = X[1];
        CKS(upload_real(x, buf));
        return spectrum_to_host(buf, out, centered);
    }

    int result_to_spectrum() override {
        if (!vol_set || !result_valid) return fail(CM_ERR_STATE, "no solver result resident");
        R* src = last_fista ? XF[last_iter % 2] : X[last_iter % 3];
        CKS(spectrum_of(src));
        CKS(launch_z<ZM_FWD>(nullptr, nullptr));
        return CM_OK;
    }

    int fsc_with(ImplBase* other_base, double* curve) override {
        auto* other = dynamic_cast<Impl*>(other_base);
        if (!other) return fail(CM_ERR_GRID_MISMATCH, "fsc: contexts differ in side or precision");
        CKS(other->result_to_spectrum());
        CK(cudaStreamSynchronize(other->stream));
        CKS(result_to_spectrum());
        const int ns = Nh + 1;
        const int blocks = 148 * 2;
        double* part = stage;                     // [blocks][ns][3] (stage holds >= 3L doubles)
        double* sums = stage + (size_t)blocks * 3 * ns;
        fsc_shell_kernel<R><<<blocks, 256, sizeof(double) * 3 * ns, stream>>>(N, S, other->S, part);
        CK(cudaGetLastError());
        fsc_reduce_kernel<<<grid_for((size_t)3 * ns, 256), 256, 0, stream>>>(part, blocks, 3 * ns, sums);
        CK(cudaGetLastError());
        std::vector<double> h((size_t)3 * ns);
        CK(cudaMemcpyAsync(h.data(), sums, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        for (int r = 0; r < ns; ++r) {
            const double den = std::sqrt(h[3 * r + 1] * h[3 * r + 2]);
            curve[r] = den > 0.0 ? h[3 * r] / den : 0.0;  // fsc.cpp:36-39
        }
        return CM_OK;
    }

    const double* result_spectrum_device(int centered) override {
        if (!vol_set || !result_valid) return nullptr;
        if (result_to_spectrum() != CM_OK) return nullptr;
        unpack_full_kernel<R><<<grid_for(L, 256), 256, 0, stream>>>(N, S, stage, centered);
        return cudaGetLastError() == cudaSuccess ? stage : nullptr;
    }

    int result_spectrum(double* out, int centered) override {
        if (!vol_set || !result_valid) return fail(CM_ERR_STATE, "no solver result resident");
        R* src = last_fista ? XF[last_iter % 2] : X[last_iter % 3];
        return spectrum_to_host(src, out, centered);  // the result buffer itself is untouched
    }
};


} // namespace cm
