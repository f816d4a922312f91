/* cm_oracle — CPU restatement of the reference M-step solver.
 *
 * TEST INFRASTRUCTURE. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load this library, and only as the checker / CPU
 * baseline. The product path (paper_1905_13408_b200/) never links it.
 *
 * Every function restates one reference function in plain C, fp64,
 * full-grid complex-to-complex exactly as the reference computes it
 * (halfshifts included). File:line citations are to
 * /root/reference/proj/src/ unless stated otherwise. Parity is pinned by
 * tests/test_oracle.py against golden vectors produced by the unmodified
 * reference (oracle/_ref/libcryomap_ref.so, tests/golden/make_golden.py).
 *
 * Layout: real volumes are x-fastest, flat (k*n + j)*n + i (volume.hpp:13);
 * complex grids are interleaved (re, im) doubles in the same order.
 */
#ifndef CM_ORACLE_H
#define CM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Same leading layout as cm_reg_config (include/cm_api.h) and RegConfig
 * (regularizer.hpp:21-35). */
typedef struct {
    double alpha, beta, gamma, eps, eps_prime, mu;
    int inner_iters;
    int step_rule; /* 0 lipschitz, 1 fixed */
    double fixed_step;
    int refresh;   /* 0 per_inner, 1 per_m_step */
    int convex_mode;
} or_reg_config;

/* Status codes: identical values to cm_status in include/cm_api.h. */
enum {
    OR_OK = 0,
    OR_ERR_INVALID_ARGUMENT = 1,
    OR_ERR_GRID_MISMATCH = 2,
    OR_ERR_NON_HERMITIAN = 3,
    OR_ERR_STEP_DIVERGED = 4,
    OR_ERR_NON_POSITIVE_SCALE = 7,
    OR_ERR_NON_HERMITIAN_INPUT = 8,
};

/* gradient.cpp:7-24 (replicate boundary) */
void or_discrete_gradient(int n, const double* x, double* d1, double* d2, double* d3);
/* gradient.cpp:29-64 (replicate boundary) */
void or_gradient_adjoint(int n, const double* d1, const double* d2, const double* d3,
                         double* out);
/* regularizer.cpp:44-59 */
void or_compute_weights(int n, const double* x, double eps, double eps_prime, int convex,
                        double* w_l1, double* w_tv);
/* regularizer.cpp:61-70 (w_tv may be NULL) */
double or_smoothed_tv_value(int n, const double* x, double mu, const double* w_tv);
/* regularizer.cpp:72-85 (w_tv may be NULL) */
void or_smoothed_tv_gradient(int n, const double* x, double mu, const double* w_tv,
                             double* out);
/* fourier.cpp:59-66 (forward, unnormalised), 109 (centered) */
void or_fft3(int n, const double* x, double* out_c);
void or_fft3_centered(int n, const double* x, double* out_c);
/* fourier.cpp:88-97 */
void or_halfshift3(int n, const double* x, double* out);
/* backproject.cpp:103-118 */
double or_symmetry_residue(int n, const double* weight, const double* num_c);
/* regularizer.cpp:87-101 */
int or_data_gradient(int n, const double* weight, const double* num_c, int finalized,
                     const double* x, double* out);
/* regularizer.cpp:103-110 */
void or_prox_l1(int n, const double* x, const double* t, double* out);
/* regularizer.cpp:33-42 */
int or_validate_reg_config(const or_reg_config* c);
/* regularizer.cpp:153-162 -> 125-149; out7 = fit,l1,tv_smooth,tv_linear,
 * restraint,lognorm_l1,lognorm_tv (regularizer.hpp:67-79) */
int or_penalized_objective(int n, const double* weight, const double* num_c, int finalized,
                           const double* x, const or_reg_config* c, const double* anchor,
                           const double* wsrc, double* out7);
/* regularizer.cpp:164-220. trace: inner_iters x 15 doubles (may be NULL);
 * *rows = rows written. */
int or_m_step(int n, const double* weight, const double* num_c, int finalized,
              const double* x_init, const double* x_anchor, const or_reg_config* c,
              double* x_out, double* trace, int* rows);
/* params.cpp:9-26 */
int or_scale_data(int n, const double* weight, const double* num_c, int finalized,
                  double* s_y, double* s_n);
/* params.cpp:40-64 */
int or_derive_config(double s_y, double s_n, double eps, double eps_prime, double a, double b,
                     double g, or_reg_config* out);

#ifdef __cplusplus
}
#endif
#endif
