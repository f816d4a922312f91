/* cm_api.h — C ABI of the B200-native M-step solver (libcm.so).
 *
 * This is the drop-in boundary for the reference's hot path,
 * cryomap::m_step (/root/reference/proj/include/cryomap/regularizer.hpp:98-100,
 * src/regularizer.cpp:164-220) and the component entry points of the same
 * header (regularizer.hpp:45-85), fourier.hpp:11-31 and params.hpp:22,39-41.
 * Plain pointers and sizes only; no exceptions cross it. Every function
 * returns a cm_status; cm_last_error() holds a thread-local message.
 *
 * Data layout (identical to the reference, volume.hpp:13-27,
 * backproject.hpp:15-25):
 *   real volume        double[n*n*n], x fastest: flat (k*n + j)*n + i
 *   accumulator weight double[n*n*n], full Fourier grid, storage indices
 *   numerator          double[2*n*n*n], interleaved (re, im), same order
 * Status codes map 1:1 to the reference exception types (errors.hpp:7-30);
 * the C++ adapter (paper_1905_13408_b200/adapter/) rethrows them.
 *
 * Threading: one context per host thread; a context is not thread-safe.
 * Calls are stream-ordered and synchronous on return. A context keeps the
 * accumulator and volumes resident in HBM between calls (em_refine calls
 * m_step once per half-map per EM iteration, refine.cpp:181,249).
 */
#ifndef CM_API_H
#define CM_API_H

#ifdef __cplusplus
extern "C" {
#endif

#define CM_API_VERSION 1

typedef enum {
    CM_OK = 0,
    CM_ERR_INVALID_ARGUMENT = 1,   /* cryomap::InvalidArgument   (regularizer.cpp:33-42) */
    CM_ERR_GRID_MISMATCH = 2,      /* cryomap::GridMismatch      (regularizer.cpp:88,169-170) */
    CM_ERR_NON_HERMITIAN = 3,      /* cryomap::NonHermitianAccumulator (regularizer.cpp:26-29) */
    CM_ERR_STEP_DIVERGED = 4,      /* cryomap::StepDiverged      (regularizer.cpp:210-213) */
    CM_ERR_CUDA = 5,               /* device / runtime failure */
    CM_ERR_NCCL = 6,               /* collective failure (multi-GPU) */
    CM_ERR_NON_POSITIVE_SCALE = 7, /* cryomap::NonPositiveScale  (params.cpp:48-50) */
    CM_ERR_NON_HERMITIAN_INPUT = 8,/* cryomap::NonHermitianInput (fourier.cpp:80-82) */
    CM_ERR_UNSUPPORTED = 9,        /* side length without a compiled radix plan */
    CM_ERR_STATE = 10,             /* call order (e.g. solve before set_accumulator) */
    CM_ERR_IO = 11,                /* cryomap::IoError           (mrc.cpp:125, 159) */
    CM_ERR_TRUNCATED_FILE = 12,    /* cryomap::TruncatedFile     (mrc.cpp:163, 184) */
    CM_ERR_BAD_MAGIC = 13,         /* cryomap::BadMagic          (mrc.cpp:166) */
    CM_ERR_UNSUPPORTED_MODE = 14   /* cryomap::UnsupportedMode   (mrc.cpp:169) */
} cm_status;

typedef struct cm_ctx cm_ctx;

/* RegConfig (regularizer.hpp:21-35) field for field, then opt-in extensions.
 * All-zero extensions reproduce the reference exactly (ISTA, exactly
 * inner_iters iterations, 1e-9 relative audit slack). */
typedef struct {
    double alpha, beta, gamma;   /* L1 / TV / restraint weights */
    double eps, eps_prime, mu;   /* reweighting offsets, TV smoothing */
    int inner_iters;
    int step_rule;               /* 0 lipschitz, 1 fixed */
    double fixed_step;
    int refresh;                 /* 0 per_inner, 1 per_m_step */
    int convex_mode;
    /* ---- extensions ---- */
    int momentum;                /* 0 ISTA (reference), 1 FISTA (no monotone audit),
                                    2 FISTA with gradient-based adaptive restart
                                    (O'Donoghue & Candes: the momentum restarts when
                                    (y_k - x_{k+1}) . (x_{k+1} - x_k) > 0) */
    int tol_kind;                /* 0 none, 1 frozen-weight surrogate relative decrease,
                                    2 step norm ||x+ - x|| relative to the largest step
                                      so far (works with FISTA) */
    double tol;                  /* stop when the measure drops below tol */
    double audit_slack;          /* <= 0: 1e-9 in fp64 (reference), 1e-6 in fp32 */
} cm_reg_config;

/* ObjectiveValue (regularizer.hpp:67-79) order:
 * fit, l1, tv_smooth, tv_linear, restraint, lognorm_l1, lognorm_tv */
typedef struct {
    double before[7];
    double after[7];
    double step;
} cm_trace_row; /* MStepTraceRow (regularizer.hpp:88-92) */

typedef struct {
    int iterations;     /* iterations behind the returned volume */
    int trace_rows;     /* rows written to trace */
    int stop_reason;    /* 1 inner_iters reached, 2 tolerance, 3 diverged */
    int diverged_iter;  /* -1 unless stop_reason == 3 */
    double last_rel;    /* last tolerance measure */
    double step;        /* l_r used */
    double solve_ms;    /* device time of the iteration loop (CUDA events) */
    int kernel_launches;/* kernels launched by the solve */
} cm_solve_stats;

int cm_version(void);
const char* cm_last_error(void);

/* Side lengths with a compiled plan (build.py SIDES): the even 2^a 3^b 5^c 7^d
 * sides 4 .. 1280 listed there (e.g. 64 100 128 160 200 256 320 360 384 400 512
 * 640 720 768 800 960 1024 1152 1200 1280); cm_last_error() after a 0 names why
 * a side is missing (odd, prime factor >= 11, above 1280, or not compiled).
 * precision: 32 (fp32 product mode) or 64 (fp64 parity mode). devices/ndev:
 * ndev == 1 is one context on one GPU; ndev > 1 shards the volume in z slabs
 * over the listed devices (cm_ctx_info, cm_set_accumulator, cm_scale_data,
 * cm_set_volumes, cm_solve, cm_get_volume and cm_m_step; the other entry points
 * return CM_ERR_UNSUPPORTED on such a context). */
int cm_supported_side(int n);
int cm_ctx_create(int n, const int* devices, int ndev, int precision, cm_ctx** out);
int cm_ctx_destroy(cm_ctx* ctx);
int cm_ctx_info(const cm_ctx* ctx, int* n, int* precision, long long* device_bytes);

/* AccumulatorPair upload (backproject.hpp:15-25): symmetry residue
 * (backproject.cpp:103-118), Hermitian projection to the packed half
 * spectrum, (-1)^(a+b+c) phase sign, max weight, data scales. */
int cm_set_accumulator(cm_ctx* ctx, const double* weight, const double* numerator,
                       int finalized);
int cm_accumulator_info(const cm_ctx* ctx, double* residue, double* max_weight);
/* scale_data (params.cpp:9-26): s_y = RMS(Re ifft3(num/sqrt(weight))), s_n = mean weight */
int cm_scale_data(cm_ctx* ctx, double* s_y, double* s_n);
/* derive_config (params.cpp:40-64); out gets RegConfig defaults elsewhere */
int cm_derive_config(double s_y, double s_n, double eps, double eps_prime, double a, double b,
                     double g, cm_reg_config* out);

/* x_init / x_anchor upload; passing the same pointer marks them as one object
 * (em_refine passes x for both, refine.cpp:181). */
int cm_set_volumes(cm_ctx* ctx, const double* x_init, const double* x_anchor);
/* Run the solver on the resident accumulator and volumes. trace may be null;
 * otherwise it receives up to trace_cap rows. */
int cm_solve(cm_ctx* ctx, const cm_reg_config* cfg, cm_trace_row* trace, int trace_cap,
             cm_solve_stats* stats);
int cm_get_volume(cm_ctx* ctx, double* x_out);
/* The spectrum of the resident solve result on the full complex grid (2*L
 * interleaved doubles): centered=1 gives fft3_centered(x) (fourier.cpp:109),
 * the V that em_refine computes after every m_step (refine.cpp:182) — here on
 * the device, from the transforms the solver already owns; centered=0 gives
 * fft3(x). The result volume stays resident. */
int cm_get_spectrum(cm_ctx* ctx, int centered, double* out_interleaved);
/* MRC volume I/O on the resident volumes (mrc.hpp:28-41):
 * mode-2 float32 x-fastest payloads are the device layout, so the files are
 * read into pinned memory and copied to the device without an fp64 detour.
 * cm_set_volumes_mrc: x_init (and x_anchor; NULL or the same path: one object)
 * from files written by write_mrc (or any conforming subset file), with the
 * reference reader's checks and error types. cm_write_volume_mrc: the resident
 * solve result, byte-identical to write_mrc(path, Volume3D(result, voxel_size)). */
int cm_set_volumes_mrc(cm_ctx* ctx, const char* path_init, const char* path_anchor);
int cm_write_volume_mrc(cm_ctx* ctx, const char* path, double voxel_size);
/* FSC (fsc.cpp:10-42) between the resident results of two contexts on the same
 * device (the two half-maps of em_refine, refine.cpp:194: fsc(V_a, V_b) with
 * V = fft3_centered(x)); curve receives n/2 + 1 shell values (cap >= n/2 + 1).
 * Both results stay resident. */
int cm_fsc(cm_ctx* a, cm_ctx* b, double* curve, int cap);

/* Backprojection: backproject_accumulate
 * (backproject.hpp:26-30, backproject.cpp:12-101) on the device, Friedel
 * finalize included, straight into the context's resident accumulator (as if
 * cm_set_accumulator(weight, numerator, finalized=1) had been called), so the
 * M-step that follows needs no upload. weight_out / numerator_out (L doubles /
 * L complex interleaved, AccumulatorPair layout) receive a copy when non-NULL.
 * The flat input mirrors ParticleSet, the PosteriorRow list and
 * OrientationGrid: */
typedef struct {
    int n_images;
    const double* images;   /* [n_images][n*n] complex interleaved: ParticleImage::f */
    const double* image_params; /* [n_images][6]: voltage_kv, defocus_A, cs_mm,
                                   amplitude_contrast, identity_flag (0/1), voxel_size */
    int n_poses;
    const double* poses;    /* [n_poses][3]: rot, tilt, psi (degrees), pose.hpp:10 */
    int n_shifts;
    const int* shifts;      /* [n_shifts][2]: dx, dy (orientation.hpp:17) */
    long long n_entries;    /* the rows' (candidate, posterior) entries, flattened */
    const long long* entry_particle;
    const unsigned* entry_candidate; /* pose * n_shifts + shift */
    const double* entry_posterior;   /* entries <= 0 are skipped (backproject.cpp:43) */
    int kernel_kind;        /* KernelKind: 0 gaussian, 1 trilinear (kernel.hpp:6) */
    double bandwidth;       /* gaussian only; must be > 0 (kernel.cpp:7-10) */
    double radius_cutoff;   /* < 0: the full plane (backproject.cpp:20) */
} cm_bp_input;
int cm_backproject(cm_ctx* ctx, const cm_bp_input* in, double* weight_out,
                   double* numerator_out);

/* E-step: e_step (estep.hpp:44-54, estep.cpp:64-270) on
 * the device. posterior receives the dense [n_images][n_poses * n_shifts]
 * matrix: row i holds PosteriorRow i's entries at their candidate indices
 * (pose * n_shifts + shift) and exact zeros elsewhere (pruned candidates),
 * each row summing to 1. volume NULL: V = fft3_centered of the context's
 * resident solve result (the M-step -> E-step hand-off of em_refine,
 * refine.cpp:182 -> 150, with no V transfer). */
typedef struct {
    int n_images;
    const double* images;       /* as cm_bp_input */
    const double* image_params; /* as cm_bp_input */
    int n_poses;
    const double* poses;        /* [n_poses][3] */
    int n_shifts;
    const int* shifts;          /* [n_shifts][2]; must include (0, 0) */
    int kernel_kind;
    double bandwidth;
    double radius_cutoff;       /* < 0: Nyquist (estep.cpp:14-17) */
    int n_sigma2;
    const double* sigma2;       /* NoiseSpectrum::sigma2, per 2D shell */
    double prune_floor;         /* estep.hpp:52 default 1e-8 */
    const double* volume;       /* FourierVolume [n^3] complex interleaved, or NULL */
} cm_estep_input;
int cm_estep(cm_ctx* ctx, const cm_estep_input* in, double* posterior);
/* The same posteriors as sparse PosteriorRow lists (estep.hpp:30-34, the
 * reference's e_step return value): row i's entries are candidate[k],
 * weight[k] for row_ptr[i] <= k < row_ptr[i+1], in ascending candidate order.
 * row_ptr has n_images + 1 slots; candidate / weight hold `capacity` entries.
 * *nnz = entries written, or, with CM_ERR_INVALID_ARGUMENT when capacity is
 * too small, the entries needed (call again with that capacity). Particles
 * are processed in device-memory-bounded batches (CM_ESTEP_BATCH_BYTES,
 * default 1 GiB), so the posterior never exists densely anywhere. */
int cm_estep_sparse(cm_ctx* ctx, const cm_estep_input* in, long long* row_ptr, int* candidate,
                    double* weight, long long capacity, long long* nnz);

/* Particle images resident on the device across EM iterations: after
 * cm_set_particles, a cm_bp_input / cm_estep_input with images == NULL (and
 * image_params == NULL) and the same n_images reads the resident set, so an
 * EM iteration moves no image data. Replaces any previous set. */
int cm_set_particles(cm_ctx* ctx, int n_images, const double* images, const double* image_params);

/* Diagnostics: when on, cm_solve launches every kernel individually between
 * CUDA events on the context stream (no graph) and accumulates per-kernel
 * device time, ms7 = {z pass (tile + column-0 kernels), y inverse, x C2R,
 * stencil sweep, finalize, x R2C, y forward}. */
int cm_set_profiling(cm_ctx* ctx, int on);
int cm_get_profile(const cm_ctx* ctx, double* ms7, int* iters);

/* m_step (regularizer.hpp:98-100) in one call: upload, solve, download. */
int cm_m_step(cm_ctx* ctx, const double* weight, const double* numerator, int finalized,
              const double* x_init, const double* x_anchor, const cm_reg_config* cfg,
              double* x_out, cm_trace_row* trace, int trace_cap, cm_solve_stats* stats);

/* ---- component entry points (regularizer.hpp:45-85, fourier.hpp) ---- */
/* data_gradient (regularizer.hpp:62) against the resident accumulator */
int cm_data_gradient(cm_ctx* ctx, const double* x, double* out);
/* compute_weights (regularizer.hpp:45-46) */
int cm_compute_weights(cm_ctx* ctx, const double* x, double eps, double eps_prime, int convex,
                       double* w_l1, double* w_tv);
/* smoothed_tv_value / smoothed_tv_gradient (regularizer.hpp:51-57); w_tv may be null */
int cm_smoothed_tv_value(cm_ctx* ctx, const double* x, double mu, const double* w_tv,
                         double* out);
int cm_smoothed_tv_gradient(cm_ctx* ctx, const double* x, double mu, const double* w_tv,
                            double* out);
/* prox_l1 (regularizer.hpp:65) */
int cm_prox_l1(cm_ctx* ctx, const double* x, const double* thresholds, double* out);
/* penalized_objective (regularizer.hpp:83-85) against the resident accumulator;
 * out7 in ObjectiveValue order */
int cm_penalized_objective(cm_ctx* ctx, const double* x, const cm_reg_config* cfg,
                           const double* x_anchor, const double* x_weights_source,
                           double* out7);
/* fft3 (fourier.hpp:11): unnormalised forward transform, full complex grid */
int cm_fft3(cm_ctx* ctx, const double* x, double* out_interleaved);
/* fft3_centered (fourier.hpp:24, fourier.cpp:109): fft3 of the half-shifted
 * volume, computed as the (-1)^(a+b+c)-signed fft3; full complex
 * grid. The resident solve result (cm_get_spectrum) is left intact. */
int cm_fft3_centered(cm_ctx* ctx, const double* x, double* out_interleaved);

/* Transform-free components for ANY side n >= 1 (the reference accepts odd and
 * tiny volumes here, test_regularizer.cpp:141-161, 245); fp64 on the current
 * device, no context. Same semantics as the context versions above. */
int cm_compute_weights_n(int n, const double* x, double eps, double eps_prime, int convex,
                         double* w_l1, double* w_tv);
int cm_smoothed_tv_value_n(int n, const double* x, double mu, const double* w_tv, double* out);
int cm_smoothed_tv_gradient_n(int n, const double* x, double mu, const double* w_tv,
                              double* out);
int cm_prox_l1_n(long long count, const double* x, const double* thresholds, double* out);

/* ---- z-slab distributed solver (one process per GPU) ----
 * The same m_step, split over `world` ranks: rank r owns the real-space planes
 * k in [r n/world, (r+1) n/world) and the spectrum rows b in the same range;
 * the transposes are NCCL all-to-alls, the stencil needs one ghost plane per
 * side. fp32, n a multiple of 128, n/world a multiple of 64.
 * nccl_id: 128 bytes from cm_nccl_unique_id on rank 0, broadcast by the caller
 * (e.g. torch.distributed); NULL emulates all `world` ranks inside this process
 * on `device` (decomposition tests on one GPU). Every rank passes the full
 * accumulator and volumes (as the reference's BackProjector state is full-grid);
 * cm_dctx_get_volume writes only the planes of the ranks this process hosts. */
typedef struct cm_dctx cm_dctx;
int cm_nccl_unique_id(unsigned char* id128);
int cm_dctx_create(int n, int world, int rank, int device, const unsigned char* nccl_id,
                   cm_dctx** out);
int cm_dctx_destroy(cm_dctx* d);
/* planes per rank, first plane of this process, ranks hosted by this process */
int cm_dctx_layout(const cm_dctx* d, int* planes_per_rank, int* first_plane, int* ranks_here);
/* Each rank uploads only the accumulator rows its b-slab reads (its spectrum
 * rows b and their mirrors N - b: about 2/P of the 24 N^3 bytes, staged from the
 * caller's pageable arrays through a pinned ring); the full-grid statistics
 * (scale_data, residue) are per-row partials all-gathered and summed in row
 * order, identical on every rank and for every P. */
int cm_dctx_set_accumulator(cm_dctx* d, const double* weight, const double* numerator,
                            int finalized);
/* host-to-device bytes of this process's last cm_dctx_set_accumulator */
int cm_dctx_upload_bytes(const cm_dctx* d, long long* acc_h2d_bytes);
int cm_dctx_set_volumes(cm_dctx* d, const double* x_init, const double* x_anchor);
int cm_dctx_solve(cm_dctx* d, const cm_reg_config* cfg, cm_trace_row* trace, int trace_cap,
                  cm_solve_stats* stats);
int cm_dctx_get_volume(cm_dctx* d, double* x_out);
/* Timing problem rendered on the device (no host copy of
 * a 1024^3 accumulator): a blob-lattice volume as x_init = x_anchor, a symmetric
 * random weight W in [1, 2) and numerator W * fft3(x) (packed column zero).
 * s_y receives the volume RMS (the derive_config input). */
int cm_dctx_set_synthetic(cm_dctx* d, unsigned long long seed, double* s_y);

#ifdef __cplusplus
}
#endif
#endif
