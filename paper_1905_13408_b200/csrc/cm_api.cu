// C ABI (include/cm_api.h) of the B200 M-step solver.
#include <cuda_runtime.h>

#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/cm_api.h"
#include "dist.cuh"
#include "impl.cuh"
#include "mrc_io.h"
#include "backproject.cuh"
#include "estep.cuh"

namespace cm {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CM_SIDES(X) X(4) X(6) X(8) X(10) X(12) X(14) X(16) X(20) X(24) X(28) X(32) X(40) X(48) \
    X(56) X(64) X(80) X(96) X(100) X(112) X(128) X(160) X(192) X(200) X(224) X(240) X(256) X(320) \
    X(360) X(384) X(400) X(448) X(480) X(512) X(640) X(720) X(768) X(800) X(960) X(1024) \
    X(1152) X(1200) X(1280)
#define CM_DECL(NN) ImplBase* make_impl_##NN(int precision);
CM_SIDES(CM_DECL)

#define CM_DDECL(NN) DistBase* make_dist_##NN();
CM_SIDES(CM_DDECL)

static DistBase* make_dist(int n) {
    switch (n) {
#define CM_DCASE(NN) \
    case NN: return make_dist_##NN();
        CM_SIDES(CM_DCASE)
#undef CM_DCASE
        default: return nullptr;
    }
}

static ImplBase* make_impl(int n, int precision) {
    switch (n) {
#define CM_CASE(NN) \
    case NN: return make_impl_##NN(precision);
        CM_SIDES(CM_CASE)
#undef CM_CASE
        default: return nullptr;
    }
}

} // namespace cm

using namespace cm;

// One context over several GPUs of the box (cm_ctx_create with ndev > 1): the
// z-slab runtime (dist.cuh) with one rank per device, each rank driven by its
// own host thread for the duration of a call (NCCL communicators of one
// process, one thread per rank: the collectives inside a solve need every rank
// running). All device ids equal: the ranks are emulated on that one GPU
// (EmuComm, device-to-device copies; the correctness configuration).
struct MultiDev {
    int n = 0, P = 0;
    std::vector<std::unique_ptr<DistBase>> ranks;  // one per device, or one hosting P virtual ranks
    template <class F> int run(F&& f) {
        const int R = (int)ranks.size();
        if (R == 1) {
            if (cudaSetDevice(ranks[0]->device) != cudaSuccess) return fail(CM_ERR_CUDA, "cudaSetDevice failed");
            return f(0, *ranks[0]);
        }
        std::vector<int> rc(R, CM_OK);
        std::vector<std::string> msg(R);
        std::vector<std::thread> th;
        for (int r = 0; r < R; ++r)
            th.emplace_back([&, r] {
                rc[r] = cudaSetDevice(ranks[r]->device) != cudaSuccess
                            ? fail(CM_ERR_CUDA, "cudaSetDevice failed")
                            : f(r, *ranks[r]);
                if (rc[r] != CM_OK) msg[r] = g_err;
            });
        for (auto& t : th) t.join();
        for (int r = 0; r < R; ++r)
            if (rc[r] != CM_OK) return fail(rc[r], "rank " + std::to_string(r) + ": " + msg[r]);
        return CM_OK;
    }
};

struct cm_ctx {
    std::unique_ptr<MultiDev> multi;  // ndev > 1
    std::unique_ptr<ImplBase> impl;
    int n = 0;
    int precision = 32;
    int device = 0;
    std::unique_ptr<MrcRing> mrc;  // pinned MRC staging, on first use
    ParticleDev particles;         // resident particle images (cm_set_particles)
};

#define CTX_GUARD(ctx)                                                         \
    do {                                                                       \
        if ((ctx) && (ctx)->multi)                                             \
            return fail(CM_ERR_UNSUPPORTED, "this entry point needs a one-GPU context (ndev == 1)"); \
        if (!(ctx) || !(ctx)->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context"); \
        if (cudaSetDevice((ctx)->device) != cudaSuccess)                       \
            return fail(CM_ERR_CUDA, "cudaSetDevice failed");                  \
    } while (0)

extern "C" {

int cm_version(void) { return CM_API_VERSION; }
const char* cm_last_error(void) { return g_err.c_str(); }

// why a side has no solver context (the reference accepts any even side through
// FFTW, volume.hpp:94-97)
static std::string unsupported_side_reason(int n) {
    const std::string sn = std::to_string(n);
    if (n < 4 || n % 2) return "side " + sn + " is not an even side >= 4 (require_even_side, volume.hpp:94-97)";
    int m = n;
    for (int p : {2, 3, 5, 7})
        while (m % p == 0) m /= p;
    if (m != 1) {
        int q = 11;
        while (m % q) q += 2;
        return "side " + sn + " has the prime factor " + std::to_string(q) +
               ": the FFT engine plans radices 2, 3, 5 and 7 only (no Bluestein stage)";
    }
    if (n > 1280)
        return "side " + sn + " exceeds 1280: N^3 >= 2^31 voxels (the kernels keep 32-bit voxel "
               "offsets) and one GPU's fp32 working set (~48 N^3 bytes) exceeds its HBM";
    return "side " + sn + " (2^a 3^b 5^c 7^d) is not among the sides compiled into this build "
           "(paper_1905_13408_b200/build.py SIDES, csrc/cm_api.cu CM_SIDES)";
}

int cm_supported_side(int n) {
    switch (n) {
#define CM_ONE(NN) case NN:
        CM_SIDES(CM_ONE)
#undef CM_ONE
        return 1;
        default:
            return 0;
    }
}

static int multi_create(int n, const int* devices, int ndev, int precision, cm_ctx** out) {
    if (!devices) return fail(CM_ERR_INVALID_ARGUMENT, "ndev > 1 needs the device list");
    if (precision != 32)
        return fail(CM_ERR_UNSUPPORTED, "multi-GPU contexts run the fp32 z-slab solver (precision 32)");
    if (n % 128 != 0 || n % ndev != 0 || (n / ndev) % 64 != 0)
        return fail(CM_ERR_UNSUPPORTED, "multi-GPU context: the z-slab solver needs n % 128 == 0 and "
                                        "n / ndev a multiple of 64 (side " + std::to_string(n) + ", " +
                                        std::to_string(ndev) + " devices)");
    bool same = true, distinct = true;
    for (int a = 0; a < ndev; ++a)
        for (int b = 0; b < ndev; ++b)
            if (a != b) {
                same &= devices[a] == devices[b];
                distinct &= devices[a] != devices[b];
            }
    if (!same && !distinct)
        return fail(CM_ERR_INVALID_ARGUMENT, "devices must be all distinct (one rank per GPU) or all "
                                             "equal (ranks emulated on one GPU)");
    auto ctx = std::make_unique<cm_ctx>();
    ctx->n = n;
    ctx->precision = precision;
    ctx->device = devices[0];
    ctx->multi = std::make_unique<MultiDev>();
    MultiDev& m = *ctx->multi;
    m.n = n;
    m.P = ndev;
    if (same) {
        CK(cudaSetDevice(devices[0]));
        m.ranks.emplace_back(make_dist(n));
        if (!m.ranks[0]) return fail(CM_ERR_UNSUPPORTED, "no z-slab build for side " + std::to_string(n));
        m.ranks[0]->device = devices[0];
        m.ranks[0]->comm = std::make_unique<EmuComm>(ndev);
        CKS(m.ranks[0]->init());
    } else {
        NcclApi& api = nccl_api();
        std::string err;
        if (!api.load(&err)) return fail(CM_ERR_NCCL, err);
        ncclUniqueId id;
        if (api.GetUniqueId(&id) != ncclSuccess) return fail(CM_ERR_NCCL, "ncclGetUniqueId failed");
        for (int r = 0; r < ndev; ++r) {
            m.ranks.emplace_back(make_dist(n));
            if (!m.ranks[r]) return fail(CM_ERR_UNSUPPORTED, "no z-slab build for side " + std::to_string(n));
            m.ranks[r]->device = devices[r];
        }
        // every rank's communicator is created concurrently (ncclCommInitRank
        // returns once all ranks have joined)
        CKS(m.run([&](int r, DistBase& d) {
            int st = 0;
            auto c = std::make_unique<NcclComm>(ndev, r, id, &st);
            if (st) return fail(CM_ERR_NCCL, "NCCL init failed: " + c->err);
            d.comm = std::move(c);
            return d.init();
        }));
    }
    *out = ctx.release();
    return CM_OK;
}

int cm_ctx_create(int n, const int* devices, int ndev, int precision, cm_ctx** out) {
    if (!out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    if (n < 4 || n % 2 != 0)
        return fail(CM_ERR_INVALID_ARGUMENT, "side_n must be even and >= 4, got " + std::to_string(n));
    if (!cm_supported_side(n)) return fail(CM_ERR_UNSUPPORTED, unsupported_side_reason(n));
    if (precision != 32 && precision != 64)
        return fail(CM_ERR_INVALID_ARGUMENT, "precision must be 32 or 64");
    if (ndev > 1) return multi_create(n, devices, ndev, precision, out);
    const int dev = (devices && ndev == 1) ? devices[0] : 0;
    CK(cudaSetDevice(dev));
    auto ctx = std::make_unique<cm_ctx>();
    ctx->n = n;
    ctx->precision = precision;
    ctx->device = dev;
    ctx->impl.reset(make_impl(n, precision));
    if (!ctx->impl) return fail(CM_ERR_UNSUPPORTED, "unsupported side");
    const int rc = ctx->impl->init();
    if (rc != CM_OK) return rc;
    *out = ctx.release();
    return CM_OK;
}

int cm_ctx_destroy(cm_ctx* ctx) {
    if (!ctx) return CM_OK;
    cudaSetDevice(ctx->device);
    delete ctx;
    return CM_OK;
}

int cm_ctx_info(const cm_ctx* ctx, int* n, int* precision, long long* device_bytes) {
    if (ctx && ctx->multi) {
        if (n) *n = ctx->n;
        if (precision) *precision = ctx->precision;
        if (device_bytes) *device_bytes = -1;
        return CM_OK;
    }
    if (!ctx || !ctx->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    if (n) *n = ctx->n;
    if (precision) *precision = ctx->precision;
    if (device_bytes) *device_bytes = ctx->impl->bytes();
    return CM_OK;
}

int cm_set_accumulator(cm_ctx* ctx, const double* weight, const double* numerator, int finalized) {
    if (ctx && ctx->multi) {
        if (!weight || !numerator) return fail(CM_ERR_INVALID_ARGUMENT, "null accumulator");
        return ctx->multi->run([&](int, DistBase& d) { return d.set_accumulator(weight, numerator, finalized); });
    }
    CTX_GUARD(ctx);
    if (!weight || !numerator) return fail(CM_ERR_INVALID_ARGUMENT, "null accumulator");
    return ctx->impl->set_accumulator(weight, numerator, finalized);
}

int cm_accumulator_info(const cm_ctx* ctx, double* residue, double* max_weight) {
    if (!ctx || !ctx->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    if (!ctx->impl->acc_set) return fail(CM_ERR_STATE, "accumulator not set");
    if (residue) *residue = ctx->impl->residue;
    if (max_weight) *max_weight = ctx->impl->max_weight;
    return CM_OK;
}

int cm_scale_data(cm_ctx* ctx, double* s_y, double* s_n) {
    if (ctx && ctx->multi) {
        DistBase& d = *ctx->multi->ranks[0];
        if (!d.acc_set) return fail(CM_ERR_STATE, "accumulator not set");
        if (!d.acc_fin) return fail(CM_ERR_NON_HERMITIAN, "scale_data: accumulator is not finalized");
        if (d.residue > 1e-8)
            return fail(CM_ERR_NON_HERMITIAN_INPUT, "ifft3: whitened accumulator is not Hermitian");
        if (s_y) *s_y = d.s_y;
        if (s_n) *s_n = d.s_n;
        return CM_OK;
    }
    CTX_GUARD(ctx);
    ImplBase* im = ctx->impl.get();
    if (!im->acc_set) return fail(CM_ERR_STATE, "accumulator not set");
    // params.cpp:10-11 checks the flag only; the Hermitian guard of ifft3
    // (fourier.cpp:80) is the symmetry residue here
    if (!im->acc_finalized)
        return fail(CM_ERR_NON_HERMITIAN, "scale_data: accumulator is not finalized");
    if (im->residue > 1e-8)
        return fail(CM_ERR_NON_HERMITIAN_INPUT, "ifft3: whitened accumulator is not Hermitian");
    if (s_y) *s_y = im->s_y;
    if (s_n) *s_n = im->s_n;
    return CM_OK;
}

int cm_derive_config(double s_y, double s_n, double eps, double eps_prime, double a, double b,
                     double g, cm_reg_config* out) {
    if (!out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    if (s_y < 0.0 || s_n < 0.0)
        return fail(CM_ERR_INVALID_ARGUMENT, "derive_config: data scales must be >= 0");
    if (!(eps > 0.0) || !(eps_prime > 0.0))
        return fail(CM_ERR_INVALID_ARGUMENT, "derive_config: eps and eps_prime must be > 0");
    if (a < 0.0 || b < 0.0 || g < 0.0)
        return fail(CM_ERR_INVALID_ARGUMENT, "derive_config: multipliers must be >= 0");
    if (s_y == 0.0 && (a > 0.0 || b > 0.0))
        return fail(CM_ERR_NON_POSITIVE_SCALE,
                    "derive_config: s_y is zero but the L1/TV multipliers are nonzero");
    std::memset(out, 0, sizeof(*out));
    out->alpha = a * s_y * eps;
    out->beta = b * s_y * eps_prime;
    out->gamma = g * s_n;
    out->eps = eps;
    out->eps_prime = eps_prime;
    out->mu = 0.01 * eps_prime;
    out->inner_iters = 24;
    return validate(out);
}

int cm_set_volumes(cm_ctx* ctx, const double* x_init, const double* x_anchor) {
    if (ctx && ctx->multi) {
        if (!x_init || !x_anchor) return fail(CM_ERR_INVALID_ARGUMENT, "null volume");
        return ctx->multi->run([&](int, DistBase& d) { return d.set_volumes(x_init, x_anchor); });
    }
    CTX_GUARD(ctx);
    if (!x_init || !x_anchor) return fail(CM_ERR_INVALID_ARGUMENT, "null volume");
    return ctx->impl->set_volumes(x_init, x_anchor);
}

int cm_solve(cm_ctx* ctx, const cm_reg_config* cfg, cm_trace_row* trace, int trace_cap,
             cm_solve_stats* stats) {
    if (ctx && ctx->multi) {
        // every rank takes the same decisions from all-reduced sums: rank 0 reports
        const int R = (int)ctx->multi->ranks.size();
        std::vector<std::vector<cm_trace_row>> tr(R);
        std::vector<cm_solve_stats> st(R);
        const int rc = ctx->multi->run([&](int r, DistBase& d) {
            if (r == 0) return d.solve(cfg, trace, trace_cap, stats ? stats : &st[0]);
            tr[r].resize(trace ? (size_t)trace_cap : 0);
            return d.solve(cfg, trace ? tr[r].data() : nullptr, trace ? trace_cap : 0, &st[r]);
        });
        return rc;
    }
    CTX_GUARD(ctx);
    return ctx->impl->solve(cfg, trace, trace_cap, stats);
}

int cm_set_profiling(cm_ctx* ctx, int on) {
    CTX_GUARD(ctx);
    ctx->impl->profiling = on;
    return CM_OK;
}

int cm_get_profile(const cm_ctx* ctx, double* ms7, int* iters) {
    if (!ctx || !ctx->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    for (int q = 0; q < 7; ++q) ms7[q] = ctx->impl->prof_ms[q];
    if (iters) *iters = ctx->impl->prof_iters;
    return CM_OK;
}

int cm_get_volume(cm_ctx* ctx, double* x_out) {
    if (ctx && ctx->multi) {
        if (!x_out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
        return ctx->multi->run([&](int, DistBase& d) { return d.get_volume(x_out); });  // disjoint planes
    }
    CTX_GUARD(ctx);
    if (!x_out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    return ctx->impl->get_volume(x_out);
}

int cm_get_spectrum(cm_ctx* ctx, int centered, double* out_interleaved) {
    CTX_GUARD(ctx);
    if (!out_interleaved) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    return ctx->impl->result_spectrum(out_interleaved, centered ? 1 : 0);
}

int cm_set_volumes_mrc(cm_ctx* ctx, const char* path_init, const char* path_anchor) {
    CTX_GUARD(ctx);
    if (!path_init) return fail(CM_ERR_INVALID_ARGUMENT, "null path");
    const bool same = !path_anchor || std::strcmp(path_init, path_anchor) == 0;
    // validate both headers before touching the resident volumes
    MrcFile fi, fa;
    size_t oi = 0, oa = 0;
    CKS(mrc_open_volume(path_init, ctx->n, fi, &oi));
    if (!same) CKS(mrc_open_volume(path_anchor, ctx->n, fa, &oa));
    if (!ctx->mrc) ctx->mrc.reset(new MrcRing());
    CKS(ctx->mrc->ensure());
    ImplBase* im = ctx->impl.get();
    const size_t L = (size_t)ctx->n * ctx->n * ctx->n;
    im->vol_set = false;  // a failed read leaves no half-set state behind
    CKS(mrc_read_payload(fi, oi, im->mrc_landing(0), L, *ctx->mrc, im->stream));
    CKS(im->mrc_commit(0));
    if (!same) {
        CKS(mrc_read_payload(fa, oa, im->mrc_landing(1), L, *ctx->mrc, im->stream));
        CKS(im->mrc_commit(1));
    } else {
        CKS(im->mrc_commit(2));
    }
    if (cudaStreamSynchronize(im->stream) != cudaSuccess)
        return fail(CM_ERR_CUDA, "mrc: upload failed");
    return CM_OK;
}

int cm_write_volume_mrc(cm_ctx* ctx, const char* path, double voxel_size) {
    CTX_GUARD(ctx);
    if (!path) return fail(CM_ERR_INVALID_ARGUMENT, "null path");
    const float* src = ctx->impl->mrc_result_f32();
    if (!src) return fail(CM_ERR_STATE, "no solver result resident");
    if (!ctx->mrc) ctx->mrc.reset(new MrcRing());
    CKS(ctx->mrc->ensure());
    return mrc_write_volume(path, ctx->n, voxel_size, src, *ctx->mrc, ctx->impl->stream);
}

int cm_backproject(cm_ctx* ctx, const cm_bp_input* in, double* weight_out, double* numerator_out) {
    CTX_GUARD(ctx);
    ImplBase* im = ctx->impl.get();
    double* stage = im->acc_stage();
    // the staging grid is scratch: the resident W / Yh (and acc_set) change only
    // in commit_acc_stage, so a call rejected by validation leaves them usable
    CKS(backproject_run(ctx->n, in, stage, im->stream, &ctx->particles));
    const size_t L = (size_t)ctx->n * ctx->n * ctx->n;
    if (weight_out &&
        cudaMemcpyAsync(weight_out, stage, sizeof(double) * L, cudaMemcpyDeviceToHost, im->stream) != cudaSuccess)
        return fail(CM_ERR_CUDA, "backproject: download failed");
    if (numerator_out && cudaMemcpyAsync(numerator_out, stage + L, sizeof(double) * 2 * L,
                                         cudaMemcpyDeviceToHost, im->stream) != cudaSuccess)
        return fail(CM_ERR_CUDA, "backproject: download failed");
    return im->commit_acc_stage(1);
}

int cm_estep(cm_ctx* ctx, const cm_estep_input* in, double* posterior) {
    CTX_GUARD(ctx);
    if (!in || !posterior) return fail(CM_ERR_INVALID_ARGUMENT, "e_step: null argument");
    const double* vdev = nullptr;
    if (!in->volume) {
        vdev = ctx->impl->result_spectrum_device(1);
        if (!vdev) return fail(CM_ERR_STATE, "e_step: no volume given and no solver result resident");
    }
    EsSink sink;
    sink.dense = posterior;
    return estep_run(ctx->n, in, in->volume, vdev, sink, ctx->impl->stream, &ctx->particles);
}

int cm_estep_sparse(cm_ctx* ctx, const cm_estep_input* in, long long* row_ptr, int* candidate,
                    double* weight, long long capacity, long long* nnz) {
    CTX_GUARD(ctx);
    if (!in || !row_ptr || !nnz || (capacity > 0 && (!candidate || !weight)))
        return fail(CM_ERR_INVALID_ARGUMENT, "e_step: null argument");
    const double* vdev = nullptr;
    if (!in->volume) {
        vdev = ctx->impl->result_spectrum_device(1);
        if (!vdev) return fail(CM_ERR_STATE, "e_step: no volume given and no solver result resident");
    }
    EsSink sink;
    sink.row_ptr = row_ptr;
    sink.cand = candidate;
    sink.weight = weight;
    sink.cap = capacity;
    const int rc = estep_run(ctx->n, in, in->volume, vdev, sink, ctx->impl->stream, &ctx->particles);
    *nnz = sink.nnz;
    return rc;
}

int cm_set_particles(cm_ctx* ctx, int n_images, const double* images, const double* image_params) {
    CTX_GUARD(ctx);
    return ctx->particles.set(ctx->n, n_images, images, image_params, ctx->impl->stream);
}

int cm_fsc(cm_ctx* a, cm_ctx* b, double* curve, int cap) {
    CTX_GUARD(a);
    if (!b || !b->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    if (!curve) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    if (a->n != b->n) return fail(CM_ERR_GRID_MISMATCH, "fsc: side_n differs");
    if (a->device != b->device) return fail(CM_ERR_INVALID_ARGUMENT, "fsc: contexts on different devices");
    if (cap < a->n / 2 + 1) return fail(CM_ERR_INVALID_ARGUMENT, "fsc: curve needs n/2 + 1 entries");
    return a->impl->fsc_with(b->impl.get(), curve);
}

int cm_m_step(cm_ctx* ctx, const double* weight, const double* numerator, int finalized,
              const double* x_init, const double* x_anchor, const cm_reg_config* cfg,
              double* x_out, cm_trace_row* trace, int trace_cap, cm_solve_stats* stats) {
    if (ctx && ctx->multi) {
        CKS(validate(cfg));
        CKS(cm_set_accumulator(ctx, weight, numerator, finalized));
        CKS(cm_set_volumes(ctx, x_init, x_anchor));
        const int rc = cm_solve(ctx, cfg, trace, trace_cap, stats);
        if (rc != CM_OK) return rc;
        return cm_get_volume(ctx, x_out);
    }
    CTX_GUARD(ctx);
    // reference order: validate config, then the accumulator guard (regularizer.cpp:167-168)
    CKS(validate(cfg));
    CKS(cm_set_accumulator(ctx, weight, numerator, finalized));
    CKS(cm_set_volumes(ctx, x_init, x_anchor));
    const int rc = cm_solve(ctx, cfg, trace, trace_cap, stats);
    if (rc != CM_OK) return rc;
    return cm_get_volume(ctx, x_out);
}

int cm_data_gradient(cm_ctx* ctx, const double* x, double* out) {
    CTX_GUARD(ctx);
    return ctx->impl->data_gradient(x, out);
}

int cm_compute_weights(cm_ctx* ctx, const double* x, double eps, double eps_prime, int convex,
                       double* w_l1, double* w_tv) {
    CTX_GUARD(ctx);
    return ctx->impl->weights(x, eps, eps_prime, convex, w_l1, w_tv);
}

int cm_smoothed_tv_value(cm_ctx* ctx, const double* x, double mu, const double* w_tv, double* out) {
    CTX_GUARD(ctx);
    return ctx->impl->tv(x, mu, w_tv, out, nullptr);
}

int cm_smoothed_tv_gradient(cm_ctx* ctx, const double* x, double mu, const double* w_tv,
                            double* out) {
    CTX_GUARD(ctx);
    return ctx->impl->tv(x, mu, w_tv, nullptr, out);
}

int cm_prox_l1(cm_ctx* ctx, const double* x, const double* thresholds, double* out) {
    CTX_GUARD(ctx);
    return ctx->impl->prox(x, thresholds, out);
}

int cm_penalized_objective(cm_ctx* ctx, const double* x, const cm_reg_config* cfg,
                           const double* x_anchor, const double* x_weights_source, double* out7) {
    CTX_GUARD(ctx);
    return ctx->impl->objective(x, cfg, x_anchor, x_weights_source, out7);
}

int cm_fft3(cm_ctx* ctx, const double* x, double* out_interleaved) {
    CTX_GUARD(ctx);
    return ctx->impl->fft3(x, out_interleaved);
}

int cm_fft3_centered(cm_ctx* ctx, const double* x, double* out_interleaved) {
    CTX_GUARD(ctx);
    if (!x || !out_interleaved) return fail(CM_ERR_INVALID_ARGUMENT, "null argument");
    return ctx->impl->fft3(x, out_interleaved, 1);
}

// ---- z-slab distributed solver ------------------------------------------------------
struct cm_dctx {
    std::unique_ptr<DistBase> impl;
    int n = 0;
};

int cm_nccl_unique_id(unsigned char* id128) {
    if (!id128) return fail(CM_ERR_INVALID_ARGUMENT, "null id");
    std::string err;
    if (!nccl_api().load(&err)) return fail(CM_ERR_NCCL, err);
    ncclUniqueId id;
    if (nccl_api().GetUniqueId(&id) != ncclSuccess) return fail(CM_ERR_NCCL, "ncclGetUniqueId failed");
    std::memcpy(id128, id.internal, sizeof(id.internal));
    return CM_OK;
}

int cm_dctx_create(int n, int world, int rank, int device, const unsigned char* nccl_id,
                   cm_dctx** out) {
    if (!out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world)
        return fail(CM_ERR_INVALID_ARGUMENT, "bad world/rank");
    if (n % 128 != 0 || n % world != 0 || (n / world) % 64 != 0)
        return fail(CM_ERR_UNSUPPORTED, "z-slab solver needs n % 128 == 0 and n/world % 64 == 0");
    CK(cudaSetDevice(device));
    auto d = std::make_unique<cm_dctx>();
    d->n = n;
    d->impl.reset(make_dist(n));
    if (!d->impl) return fail(CM_ERR_UNSUPPORTED, "no z-slab build for side " + std::to_string(n));
    d->impl->device = device;
    if (nccl_id) {
        ncclUniqueId id;
        std::memcpy(id.internal, nccl_id, sizeof(id.internal));
        int st = 0;
        auto c = std::make_unique<NcclComm>(world, rank, id, &st);
        if (st) return fail(CM_ERR_NCCL, "NCCL init failed: " + c->err);
        d->impl->comm = std::move(c);
    } else {
        if (rank != 0) return fail(CM_ERR_INVALID_ARGUMENT, "emulated ranks: pass rank 0");
        d->impl->comm = std::make_unique<EmuComm>(world);
    }
    const int rc = d->impl->init();
    if (rc != CM_OK) return rc;
    *out = d.release();
    return CM_OK;
}

#define DCTX_GUARD(d)                                                                      \
    do {                                                                                   \
        if (!(d) || !(d)->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");      \
        if (cudaSetDevice((d)->impl->device) != cudaSuccess)                               \
            return fail(CM_ERR_CUDA, "cudaSetDevice failed");                              \
    } while (0)

int cm_dctx_destroy(cm_dctx* d) {
    if (!d) return CM_OK;
    if (d->impl) cudaSetDevice(d->impl->device);
    delete d;
    return CM_OK;
}

int cm_dctx_layout(const cm_dctx* d, int* planes_per_rank, int* first_plane, int* ranks_here) {
    if (!d || !d->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    const Comm& c = *d->impl->comm;
    if (planes_per_rank) *planes_per_rank = d->n / c.P;
    if (first_plane) *first_plane = c.rank0 * (d->n / c.P);
    if (ranks_here) *ranks_here = c.nv;
    return CM_OK;
}

int cm_dctx_upload_bytes(const cm_dctx* d, long long* acc_h2d_bytes) {
    if (!d || !d->impl) return fail(CM_ERR_INVALID_ARGUMENT, "null context");
    if (acc_h2d_bytes) *acc_h2d_bytes = (long long)d->impl->acc_h2d_bytes;
    return CM_OK;
}

int cm_dctx_set_accumulator(cm_dctx* d, const double* weight, const double* numerator,
                            int finalized) {
    DCTX_GUARD(d);
    if (!weight || !numerator) return fail(CM_ERR_INVALID_ARGUMENT, "null accumulator");
    return d->impl->set_accumulator(weight, numerator, finalized);
}

int cm_dctx_set_volumes(cm_dctx* d, const double* x_init, const double* x_anchor) {
    DCTX_GUARD(d);
    if (!x_init || !x_anchor) return fail(CM_ERR_INVALID_ARGUMENT, "null volume");
    return d->impl->set_volumes(x_init, x_anchor);
}

int cm_dctx_solve(cm_dctx* d, const cm_reg_config* cfg, cm_trace_row* trace, int trace_cap,
                  cm_solve_stats* stats) {
    DCTX_GUARD(d);
    return d->impl->solve(cfg, trace, trace_cap, stats);
}

int cm_dctx_get_volume(cm_dctx* d, double* x_out) {
    DCTX_GUARD(d);
    if (!x_out) return fail(CM_ERR_INVALID_ARGUMENT, "null out");
    return d->impl->get_volume(x_out);
}

int cm_dctx_set_synthetic(cm_dctx* d, unsigned long long seed, double* s_y) {
    DCTX_GUARD(d);
    return d->impl->set_synthetic(seed, s_y);
}

} // extern "C"
