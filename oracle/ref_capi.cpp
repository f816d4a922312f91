// C entry points over the UNMODIFIED reference library — TEST INFRASTRUCTURE.
//
// Compiled by oracle/Makefile together with /root/reference/proj/src/*.cpp
// into oracle/_ref/libcryomap_ref.so. Only tests/ (golden-fixture
// generation), __graft_entry__.smoke() (never) and bench.py's reference arm /
// cpu_baseline leg load it. Every function converts plain buffers into the
// reference's own types and calls the reference's public API:
//   m_step                    regularizer.hpp:98-100
//   data_gradient             regularizer.hpp:62
//   penalized_objective       regularizer.hpp:83-85
//   compute_weights           regularizer.hpp:45-46
//   smoothed_tv_value/grad    regularizer.hpp:51-57
//   prox_l1                   regularizer.hpp:65
//   scale_data/derive_config  params.hpp:22, 39-41
//   fft3 / ifft3_complex      fourier.hpp:11-18
//   accumulator_symmetry_residue backproject.hpp:35
//   fsc of fft3_centered volumes fsc.hpp:21 (em_refine, refine.cpp:194)
// Errors are mapped to the same status codes as include/cm_api.h.
#include <chrono>
#include <complex>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "cryomap/backproject.hpp"
#include "cryomap/estep.hpp"
#include "cryomap/fourier.hpp"
#include "cryomap/fsc.hpp"
#include "cryomap/gradient.hpp"
#include "cryomap/mrc.hpp"
#include "cryomap/orientation.hpp"
#include "cryomap/params.hpp"
#include "cryomap/phantom.hpp"
#include "cryomap/regularizer.hpp"

using namespace cryomap;

namespace {

thread_local std::string g_err;

enum {
    REF_OK = 0,
    REF_ERR_INVALID_ARGUMENT = 1,
    REF_ERR_GRID_MISMATCH = 2,
    REF_ERR_NON_HERMITIAN = 3,
    REF_ERR_STEP_DIVERGED = 4,
    REF_ERR_NON_POSITIVE_SCALE = 7,
    REF_ERR_NON_HERMITIAN_INPUT = 8,
    REF_ERR_IO = 11,
    REF_ERR_TRUNCATED_FILE = 12,
    REF_ERR_BAD_MAGIC = 13,
    REF_ERR_UNSUPPORTED_MODE = 14,
    REF_ERR_OTHER = 99,
};

template <typename F>
int guard(F&& f) {
    try {
        f();
        return REF_OK;
    } catch (const InvalidArgument& e) {
        g_err = e.what();
        return REF_ERR_INVALID_ARGUMENT;
    } catch (const GridMismatch& e) {
        g_err = e.what();
        return REF_ERR_GRID_MISMATCH;
    } catch (const NonHermitianAccumulator& e) {
        g_err = e.what();
        return REF_ERR_NON_HERMITIAN;
    } catch (const StepDiverged& e) {
        g_err = e.what();
        return REF_ERR_STEP_DIVERGED;
    } catch (const NonPositiveScale& e) {
        g_err = e.what();
        return REF_ERR_NON_POSITIVE_SCALE;
    } catch (const NonHermitianInput& e) {
        g_err = e.what();
        return REF_ERR_NON_HERMITIAN_INPUT;
    } catch (const IoError& e) {
        g_err = e.what();
        return REF_ERR_IO;
    } catch (const TruncatedFile& e) {
        g_err = e.what();
        return REF_ERR_TRUNCATED_FILE;
    } catch (const BadMagic& e) {
        g_err = e.what();
        return REF_ERR_BAD_MAGIC;
    } catch (const UnsupportedMode& e) {
        g_err = e.what();
        return REF_ERR_UNSUPPORTED_MODE;
    } catch (const std::exception& e) {
        g_err = e.what();
        return REF_ERR_OTHER;
    }
}

// Mirrors cm_reg_config's leading fields (include/cm_api.h).
struct RefRegConfig {
    double alpha, beta, gamma, eps, eps_prime, mu;
    int inner_iters;
    int step_rule; // 0 lipschitz, 1 fixed
    double fixed_step;
    int refresh;   // 0 per_inner, 1 per_m_step
    int convex_mode;
};

RegConfig to_reg(const RefRegConfig* c) {
    RegConfig r;
    r.alpha = c->alpha;
    r.beta = c->beta;
    r.gamma = c->gamma;
    r.eps = c->eps;
    r.eps_prime = c->eps_prime;
    r.mu = c->mu;
    r.inner_iters = c->inner_iters;
    r.step_rule = c->step_rule == 1 ? RegConfig::StepRule::fixed : RegConfig::StepRule::lipschitz;
    r.fixed_step = c->fixed_step;
    r.refresh = c->refresh == 1 ? RegConfig::Refresh::per_m_step : RegConfig::Refresh::per_inner;
    r.convex_mode = c->convex_mode != 0;
    return r;
}

Volume3D to_vol(int n, const double* x) {
    Volume3D v(n, 1.0);
    std::memcpy(v.data.data(), x, sizeof(double) * v.data.size());
    return v;
}

AccumulatorPair to_acc(int n, const double* w, const double* y, int finalized) {
    AccumulatorPair a;
    a.side_n = n;
    a.voxel_size = 1.0;
    const std::size_t L = std::size_t(n) * n * n;
    a.weight.assign(w, w + L);
    a.numerator.resize(L);
    std::memcpy(reinterpret_cast<double*>(a.numerator.data()), y, sizeof(double) * 2 * L);
    a.finalized = finalized != 0;
    return a;
}

void put_obj(const ObjectiveValue& o, double* out) {
    out[0] = o.fit;
    out[1] = o.l1;
    out[2] = o.tv_smooth;
    out[3] = o.tv_linear;
    out[4] = o.restraint;
    out[5] = o.lognorm_l1;
    out[6] = o.lognorm_tv;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// trace: inner_iters rows x 15 doubles (before[7], after[7], step), may be
// null. *rows receives the number of trace rows written (also on error).
// *seconds receives the wall time of the m_step call alone.
int ref_m_step(int n, const double* weight, const double* numerator, int finalized,
               const double* x_init, const double* x_anchor, const RefRegConfig* cfg,
               double* x_out, double* trace, int* rows, double* seconds) {
    std::vector<MStepTraceRow> tr;
    int rc = guard([&] {
        AccumulatorPair acc = to_acc(n, weight, numerator, finalized);
        Volume3D xi = to_vol(n, x_init);
        Volume3D xa = to_vol(n, x_anchor);
        RegConfig rc2 = to_reg(cfg);
        auto t0 = std::chrono::steady_clock::now();
        Volume3D out = m_step(acc, xi, xa, rc2, trace ? &tr : nullptr);
        auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        std::memcpy(x_out, out.data.data(), sizeof(double) * out.data.size());
    });
    if (rows) *rows = int(tr.size());
    if (trace)
        for (std::size_t r = 0; r < tr.size(); ++r) {
            put_obj(tr[r].before, trace + 15 * r);
            put_obj(tr[r].after, trace + 15 * r + 7);
            trace[15 * r + 14] = tr[r].step;
        }
    return rc;
}

int ref_data_gradient(int n, const double* weight, const double* numerator, int finalized,
                      const double* x, double* out) {
    return guard([&] {
        AccumulatorPair acc = to_acc(n, weight, numerator, finalized);
        Volume3D g = data_gradient(to_vol(n, x), acc);
        std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
    });
}

int ref_penalized_objective(int n, const double* weight, const double* numerator,
                            int finalized, const double* x, const RefRegConfig* cfg,
                            const double* anchor, const double* wsrc, double* out7) {
    return guard([&] {
        AccumulatorPair acc = to_acc(n, weight, numerator, finalized);
        ObjectiveValue o = penalized_objective(to_vol(n, x), acc, to_reg(cfg),
                                               to_vol(n, anchor), to_vol(n, wsrc));
        put_obj(o, out7);
    });
}

int ref_compute_weights(int n, const double* x, double eps, double eps_prime, int convex,
                        double* w_l1, double* w_tv) {
    return guard([&] {
        WeightFields w = compute_weights(to_vol(n, x), eps, eps_prime, convex != 0);
        std::memcpy(w_l1, w.w_l1.data(), sizeof(double) * w.w_l1.size());
        std::memcpy(w_tv, w.w_tv.data(), sizeof(double) * w.w_tv.size());
    });
}

int ref_smoothed_tv_value(int n, const double* x, double mu, const double* w_tv,
                          double* out) {
    return guard([&] {
        std::vector<double> w;
        if (w_tv) w.assign(w_tv, w_tv + std::size_t(n) * n * n);
        *out = smoothed_tv_value(to_vol(n, x), mu, w_tv ? &w : nullptr);
    });
}

int ref_smoothed_tv_gradient(int n, const double* x, double mu, const double* w_tv,
                             double* out) {
    return guard([&] {
        std::vector<double> w;
        if (w_tv) w.assign(w_tv, w_tv + std::size_t(n) * n * n);
        Volume3D g = smoothed_tv_gradient(to_vol(n, x), mu, w_tv ? &w : nullptr);
        std::memcpy(out, g.data.data(), sizeof(double) * g.data.size());
    });
}

int ref_prox_l1(int n, const double* x, const double* t, double* out) {
    return guard([&] {
        Volume3D v = to_vol(n, x);
        std::vector<double> th(t, t + v.data.size());
        Volume3D o = prox_l1(v, th);
        std::memcpy(out, o.data.data(), sizeof(double) * o.data.size());
    });
}

int ref_discrete_gradient(int n, const double* x, double* d1, double* d2, double* d3) {
    return guard([&] {
        GradientField g = discrete_gradient(to_vol(n, x));
        std::memcpy(d1, g.d1.data(), sizeof(double) * g.d1.size());
        std::memcpy(d2, g.d2.data(), sizeof(double) * g.d2.size());
        std::memcpy(d3, g.d3.data(), sizeof(double) * g.d3.size());
    });
}

int ref_scale_data(int n, const double* weight, const double* numerator, int finalized,
                   double* s_y, double* s_n) {
    return guard([&] {
        DataScales s = scale_data(to_acc(n, weight, numerator, finalized));
        *s_y = s.s_y;
        *s_n = s.s_n;
    });
}

int ref_derive_config(double s_y, double s_n, double eps, double eps_prime, double a,
                      double b, double g, RefRegConfig* out) {
    return guard([&] {
        RegConfig c = derive_config(s_y, s_n, eps, eps_prime, Multipliers{a, b, g});
        out->alpha = c.alpha;
        out->beta = c.beta;
        out->gamma = c.gamma;
        out->eps = c.eps;
        out->eps_prime = c.eps_prime;
        out->mu = c.mu;
        out->inner_iters = c.inner_iters;
        out->step_rule = 0;
        out->fixed_step = 0.0;
        out->refresh = 0;
        out->convex_mode = 0;
    });
}

int ref_fft3(int n, const double* x, double* out_interleaved) {
    return guard([&] {
        FourierVolume F = fft3(to_vol(n, x));
        std::memcpy(out_interleaved, reinterpret_cast<const double*>(F.data.data()),
                    sizeof(double) * 2 * F.data.size());
    });
}

int ref_fft3_centered(int n, const double* x, double* out_interleaved) {
    return guard([&] {
        FourierVolume F = fft3_centered(to_vol(n, x));
        std::memcpy(out_interleaved, reinterpret_cast<const double*>(F.data.data()),
                    sizeof(double) * 2 * F.data.size());
    });
}

int ref_symmetry_residue(int n, const double* weight, const double* numerator, double* out) {
    return guard([&] { *out = accumulator_symmetry_residue(to_acc(n, weight, numerator, 1)); });
}

// Phantom from the reference generator (phantom.hpp:23-27).
int ref_phantom(int n, int n_blobs, unsigned long long seed, double* out) {
    return guard([&] {
        Volume3D v = generate_phantom(random_phantom_spec(n_blobs, n, seed), n, 1.0);
        std::memcpy(out, v.data.data(), sizeof(double) * v.data.size());
    });
}

// FSC of two real volumes as em_refine forms it: fsc(fft3_centered(a), fft3_centered(b))
int ref_fsc_volumes(int n, const double* a, const double* b, double* curve) {
    return guard([&] {
        FSCCurve c = fsc(fft3_centered(to_vol(n, a)), fft3_centered(to_vol(n, b)));
        std::memcpy(curve, c.value.data(), sizeof(double) * c.value.size());
    });
}

// backproject_accumulate (backproject.cpp:12-101) over the flat cm_bp_input
// layout (include/cm_api.h): consecutive entries of one particle form a row.
int ref_backproject(int n, int n_images, const double* images, const double* image_params,
                    int n_poses, const double* poses, int n_shifts, const int* shifts,
                    long long n_entries, const long long* entry_particle,
                    const unsigned* entry_candidate, const double* entry_posterior,
                    int kernel_kind, double bandwidth, double radius_cutoff, int threads,
                    double* weight_out, double* numerator_out) {
    return guard([&] {
        ParticleSet parts;
        parts.side_n = n;
        parts.voxel_size = n_images > 0 ? image_params[5] : 1.0;
        const size_t plane = size_t(n) * n;
        for (int i = 0; i < n_images; ++i) {
            ParticleImage img;
            img.side_n = n;
            const double* ip = image_params + 6 * size_t(i);
            img.ctf.voltage_kv = ip[0];
            img.ctf.defocus_A = ip[1];
            img.ctf.cs_mm = ip[2];
            img.ctf.amplitude_contrast = ip[3];
            img.ctf.identity_flag = ip[4] != 0.0;
            img.voxel_size = ip[5];
            img.f.resize(plane);
            std::memcpy(img.f.data(), images + 2 * plane * size_t(i), sizeof(double) * 2 * plane);
            img.id = i;
            parts.items.push_back(std::move(img));
        }
        OrientationGrid grid;
        grid.side_n = n;
        for (int q = 0; q < n_poses; ++q)
            grid.poses.push_back(Pose{poses[3 * q], poses[3 * q + 1], poses[3 * q + 2], 0.0, 0.0});
        for (int q = 0; q < n_shifts; ++q) grid.shifts.emplace_back(shifts[2 * q], shifts[2 * q + 1]);
        std::vector<PosteriorRow> rows;
        for (long long e = 0; e < n_entries; ++e) {
            if (rows.empty() || rows.back().particle != size_t(entry_particle[e])) {
                rows.emplace_back();
                rows.back().particle = size_t(entry_particle[e]);
            }
            rows.back().entries.emplace_back(entry_candidate[e], entry_posterior[e]);
        }
        const KernelSpec kernel{kernel_kind == 0 ? KernelKind::gaussian : KernelKind::trilinear,
                                bandwidth};
        AccumulatorPair acc = backproject_accumulate(parts, rows, kernel, grid, radius_cutoff, threads);
        std::memcpy(weight_out, acc.weight.data(), sizeof(double) * acc.weight.size());
        std::memcpy(numerator_out, acc.numerator.data(), sizeof(double) * 2 * acc.numerator.size());
    });
}

// e_step (estep.cpp:64-270) over the flat cm_estep_input layout; the rows are
// scattered into a dense [n_images][n_poses * n_shifts] matrix
int ref_estep(int n, int n_images, const double* images, const double* image_params, int n_poses,
              const double* poses, int n_shifts, const int* shifts, int kernel_kind, double bandwidth,
              double radius_cutoff, int n_sigma2, const double* sigma2, double prune_floor,
              const double* volume, int threads, double* dense_out) {
    return guard([&] {
        ParticleSet parts;
        parts.side_n = n;
        parts.voxel_size = n_images > 0 ? image_params[5] : 1.0;
        const size_t plane = size_t(n) * n;
        for (int i = 0; i < n_images; ++i) {
            ParticleImage img;
            img.side_n = n;
            const double* ip = image_params + 6 * size_t(i);
            img.ctf.voltage_kv = ip[0];
            img.ctf.defocus_A = ip[1];
            img.ctf.cs_mm = ip[2];
            img.ctf.amplitude_contrast = ip[3];
            img.ctf.identity_flag = ip[4] != 0.0;
            img.voxel_size = ip[5];
            img.f.resize(plane);
            std::memcpy(img.f.data(), images + 2 * plane * size_t(i), sizeof(double) * 2 * plane);
            parts.items.push_back(std::move(img));
        }
        OrientationGrid grid;
        grid.side_n = n;
        for (int q = 0; q < n_poses; ++q)
            grid.poses.push_back(Pose{poses[3 * q], poses[3 * q + 1], poses[3 * q + 2], 0.0, 0.0});
        for (int q = 0; q < n_shifts; ++q) grid.shifts.emplace_back(shifts[2 * q], shifts[2 * q + 1]);
        FourierVolume V(n, parts.voxel_size);
        std::memcpy(V.data.data(), volume, sizeof(double) * 2 * V.data.size());
        NoiseSpectrum noise;
        noise.sigma2.assign(sigma2, sigma2 + n_sigma2);
        const KernelSpec kernel{kernel_kind == 0 ? KernelKind::gaussian : KernelKind::trilinear,
                                bandwidth};
        auto rows = e_step(parts, V, grid, kernel, noise, radius_cutoff, prune_floor, threads);
        const size_t nc = size_t(n_poses) * n_shifts;
        std::memset(dense_out, 0, sizeof(double) * nc * n_images);
        for (const PosteriorRow& r : rows)
            for (const auto& [c, w] : r.entries) dense_out[r.particle * nc + c] = w;
    });
}

// write_mrc(path, Volume3D) / read_mrc_volume(path) (mrc.cpp:134, 219)
int ref_write_mrc_volume(const char* path, int n, double voxel_size, const double* x) {
    return guard([&] {
        Volume3D v = to_vol(n, x);
        v.voxel_size = voxel_size;
        write_mrc(path, v);
    });
}

int ref_read_mrc_volume(const char* path, int n, double* x, double* voxel_size) {
    return guard([&] {
        Volume3D v = read_mrc_volume(path);
        if (v.side_n != n) throw GridMismatch("ref_read_mrc_volume: side differs");
        std::memcpy(x, v.data.data(), sizeof(double) * v.data.size());
        if (voxel_size) *voxel_size = v.voxel_size;
    });
}

} // extern "C"
