/* cm_oracle — CPU restatement of the reference M-step solver.
 * TEST INFRASTRUCTURE ONLY; see cm_oracle.h for the contract. */
#include "cm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "fftc.h"

static size_t vol(int n) { return (size_t)n * (size_t)n * (size_t)n; }
static size_t at(int n, int i, int j, int k) { return ((size_t)k * n + j) * n + i; }

/* ---- L1 numerics ------------------------------------------------------ */

/* Backward differences, zero on the first plane of each axis
 * (gradient.cpp:7-24, replicate branch). */
void or_discrete_gradient(int n, const double* x, double* d1, double* d2, double* d3) {
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                const size_t m = at(n, i, j, k);
                const double v = x[m];
                d1[m] = i ? v - x[at(n, i - 1, j, k)] : 0.0;
                d2[m] = j ? v - x[at(n, i, j - 1, k)] : 0.0;
                d3[m] = k ? v - x[at(n, i, j, k - 1)] : 0.0;
            }
}

/* Exact adjoint of the above (gradient.cpp:26-64): per axis the sample
 * itself enters with + unless it is on the first plane, and the forward
 * neighbour enters with - unless the sample is on the last plane. */
void or_gradient_adjoint(int n, const double* d1, const double* d2, const double* d3,
                         double* out) {
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i) {
                double s = 0.0;
                if (i > 0) s += d1[at(n, i, j, k)];
                if (i < n - 1) s -= d1[at(n, i + 1, j, k)];
                if (j > 0) s += d2[at(n, i, j, k)];
                if (j < n - 1) s -= d2[at(n, i, j + 1, k)];
                if (k > 0) s += d3[at(n, i, j, k)];
                if (k < n - 1) s -= d3[at(n, i, j, k + 1)];
                out[at(n, i, j, k)] = s;
            }
}

static double gnorm(const double* d1, const double* d2, const double* d3, size_t m) {
    return sqrt(d1[m] * d1[m] + d2[m] * d2[m] + d3[m] * d3[m]);
}

/* regularizer.cpp:12-14 */
static double huber(double g, double mu) { return g < mu ? g * g / (2.0 * mu) : g - mu / 2.0; }

void or_halfshift3(int n, const double* x, double* out) {
    const int h = n / 2;
    for (int k = 0; k < n; ++k)
        for (int j = 0; j < n; ++j)
            for (int i = 0; i < n; ++i)
                out[at(n, i, j, k)] = x[at(n, (i + h) % n, (j + h) % n, (k + h) % n)];
}

void or_fft3(int n, const double* x, double* out_c) {
    const size_t L = vol(n);
    fftc_cplx* c = (fftc_cplx*)out_c;
    for (size_t m = 0; m < L; ++m) {
        c[m].re = x[m];
        c[m].im = 0.0;
    }
    fftc_3d(c, c, n, n, n, -1);
}

void or_fft3_centered(int n, const double* x, double* out_c) {
    double* s = (double*)malloc(sizeof(double) * vol(n));
    or_halfshift3(n, x, s);
    or_fft3(n, s, out_c);
    free(s);
}

/* ---- accumulator guard (backproject.cpp:103-118) ------------------------ */

double or_symmetry_residue(int n, const double* w, const double* y) {
    double worst = 0.0, scale = 0.0;
    for (int c = 0; c < n; ++c)
        for (int b = 0; b < n; ++b)
            for (int a = 0; a < n; ++a) {
                const size_t m = at(n, a, b, c);
                const size_t q = at(n, a ? n - a : 0, b ? n - b : 0, c ? n - c : 0);
                const double dr = y[2 * m] - y[2 * q];
                const double di = y[2 * m + 1] + y[2 * q + 1];
                const double dz = sqrt(dr * dr + di * di);
                if (dz > worst) worst = dz;
                const double dw = fabs(w[m] - w[q]);
                if (dw > worst) worst = dw;
                const double az = sqrt(y[2 * m] * y[2 * m] + y[2 * m + 1] * y[2 * m + 1]);
                if (az > scale) scale = az;
                if (w[m] > scale) scale = w[m];
            }
    return scale > 0.0 ? worst / scale : 0.0;
}

static int finalized_ok(int n, const double* w, const double* y, int finalized) {
    /* regularizer.cpp:26-29 */
    return finalized && !(or_symmetry_residue(n, w, y) > 1e-9);
}

/* ---- regularizer pieces -------------------------------------------------- */

void or_compute_weights(int n, const double* x, double eps, double eps_prime, int convex,
                        double* w_l1, double* w_tv) {
    const size_t L = vol(n);
    if (convex) {
        for (size_t m = 0; m < L; ++m) w_l1[m] = w_tv[m] = 1.0;
        return;
    }
    double* d = (double*)malloc(sizeof(double) * 3 * L);
    or_discrete_gradient(n, x, d, d + L, d + 2 * L);
    for (size_t m = 0; m < L; ++m) {
        w_l1[m] = 1.0 / (fabs(x[m]) + eps);
        w_tv[m] = 1.0 / (gnorm(d, d + L, d + 2 * L, m) + eps_prime);
    }
    free(d);
}

double or_smoothed_tv_value(int n, const double* x, double mu, const double* w_tv) {
    const size_t L = vol(n);
    double* d = (double*)malloc(sizeof(double) * 3 * L);
    or_discrete_gradient(n, x, d, d + L, d + 2 * L);
    double s = 0.0;
    for (size_t m = 0; m < L; ++m) {
        const double h = huber(gnorm(d, d + L, d + 2 * L, m), mu);
        s += w_tv ? w_tv[m] * h : h;
    }
    free(d);
    return s;
}

void or_smoothed_tv_gradient(int n, const double* x, double mu, const double* w_tv,
                             double* out) {
    const size_t L = vol(n);
    double* d = (double*)malloc(sizeof(double) * 3 * L);
    or_discrete_gradient(n, x, d, d + L, d + 2 * L);
    for (size_t m = 0; m < L; ++m) {
        const double g = gnorm(d, d + L, d + 2 * L, m);
        double sc = 1.0 / (mu > g ? mu : g);
        if (w_tv) sc *= w_tv[m];
        d[m] *= sc;
        d[L + m] *= sc;
        d[2 * L + m] *= sc;
    }
    or_gradient_adjoint(n, d, d + L, d + 2 * L, out);
    free(d);
}

/* Half the gradient of the fit (regularizer.cpp:87-101): halfshift, forward
 * c2c, W*F - Y, backward c2c / L, real part, halfshift back. */
static void data_gradient_nocheck(int n, const double* w, const double* y, const double* x,
                                  double* out) {
    const size_t L = vol(n);
    fftc_cplx* F = (fftc_cplx*)malloc(sizeof(fftc_cplx) * L);
    or_fft3_centered(n, x, (double*)F);
    for (size_t m = 0; m < L; ++m) {
        F[m].re = w[m] * F[m].re - y[2 * m];
        F[m].im = w[m] * F[m].im - y[2 * m + 1];
    }
    fftc_3d(F, F, n, n, n, +1);
    double* g = (double*)malloc(sizeof(double) * L);
    const double inv = 1.0 / (double)L;
    for (size_t m = 0; m < L; ++m) g[m] = F[m].re * inv;
    or_halfshift3(n, g, out);
    free(g);
    free(F);
}

int or_data_gradient(int n, const double* w, const double* y, int finalized, const double* x,
                     double* out) {
    if (!finalized_ok(n, w, y, finalized)) return OR_ERR_NON_HERMITIAN;
    data_gradient_nocheck(n, w, y, x, out);
    return OR_OK;
}

void or_prox_l1(int n, const double* x, const double* t, double* out) {
    const size_t L = vol(n);
    for (size_t m = 0; m < L; ++m)
        out[m] = fabs(x[m]) <= t[m] ? 0.0 : x[m] - copysign(t[m], x[m]);
}

int or_validate_reg_config(const or_reg_config* c) {
    if (c->alpha < 0.0 || c->beta < 0.0 || c->gamma < 0.0) return OR_ERR_INVALID_ARGUMENT;
    if (c->eps <= 0.0 || c->eps_prime <= 0.0 || c->mu <= 0.0) return OR_ERR_INVALID_ARGUMENT;
    if (c->inner_iters < 1) return OR_ERR_INVALID_ARGUMENT;
    if (c->step_rule == 1 && c->fixed_step <= 0.0) return OR_ERR_INVALID_ARGUMENT;
    return OR_OK;
}

/* regularizer.cpp:114-123 */
static double fit_value(int n, const double* w, const double* y, const double* x) {
    const size_t L = vol(n);
    fftc_cplx* F = (fftc_cplx*)malloc(sizeof(fftc_cplx) * L);
    or_fft3_centered(n, x, (double*)F);
    double quad = 0.0, cross = 0.0;
    for (size_t m = 0; m < L; ++m) {
        quad += w[m] * (F[m].re * F[m].re + F[m].im * F[m].im);
        cross += y[2 * m] * F[m].re + y[2 * m + 1] * F[m].im;
    }
    free(F);
    return (quad - 2.0 * cross) / (double)L;
}

/* regularizer.cpp:125-149 */
static void objective_with_weights(int n, const double* w, const double* y, const double* x,
                                   const or_reg_config* c, const double* anchor,
                                   const double* w_l1, const double* w_tv, double* o) {
    const size_t L = vol(n);
    double l1 = 0, tvs = 0, tvl = 0, ln1 = 0, lntv = 0, rs = 0;
    o[0] = fit_value(n, w, y, x);
    double* d = (double*)malloc(sizeof(double) * 3 * L);
    or_discrete_gradient(n, x, d, d + L, d + 2 * L);
    for (size_t m = 0; m < L; ++m) {
        const double ax = fabs(x[m]);
        const double gn = gnorm(d, d + L, d + 2 * L, m);
        l1 += w_l1[m] * ax;
        tvs += w_tv[m] * huber(gn, c->mu);
        tvl += w_tv[m] * gn;
        ln1 += log(ax + c->eps);
        lntv += log(gn + c->eps_prime);
        const double dd = x[m] - anchor[m];
        rs += dd * dd;
    }
    free(d);
    o[1] = c->alpha * l1;
    o[2] = c->beta * tvs;
    o[3] = c->beta * tvl;
    o[4] = c->gamma * rs;
    o[5] = c->alpha * ln1;
    o[6] = c->beta * lntv;
}

static double surrogate(const double* o) { return o[0] + o[1] + o[2] + o[4]; }

int or_penalized_objective(int n, const double* w, const double* y, int finalized,
                           const double* x, const or_reg_config* c, const double* anchor,
                           const double* wsrc, double* out7) {
    int rc = or_validate_reg_config(c);
    if (rc) return rc;
    if (!finalized_ok(n, w, y, finalized)) return OR_ERR_NON_HERMITIAN;
    const size_t L = vol(n);
    double* wl = (double*)malloc(sizeof(double) * 2 * L);
    or_compute_weights(n, wsrc, c->eps, c->eps_prime, c->convex_mode, wl, wl + L);
    objective_with_weights(n, w, y, x, c, anchor, wl, wl + L, out7);
    free(wl);
    return OR_OK;
}

/* ISTA driver (regularizer.cpp:164-220). */
int or_m_step(int n, const double* w, const double* y, int finalized, const double* x_init,
              const double* x_anchor, const or_reg_config* c, double* x_out, double* trace,
              int* rows) {
    if (rows) *rows = 0;
    int rc = or_validate_reg_config(c);
    if (rc) return rc;
    if (!finalized_ok(n, w, y, finalized)) return OR_ERR_NON_HERMITIAN;
    const size_t L = vol(n);
    const int lipschitz = c->step_rule == 0;
    double maxw = 0.0;
    for (size_t m = 0; m < L; ++m)
        if (w[m] > maxw) maxw = w[m];

    double* x = (double*)malloc(sizeof(double) * L);
    double* nx = (double*)malloc(sizeof(double) * L);
    double* wl = (double*)malloc(sizeof(double) * 2 * L);
    double* g = (double*)malloc(sizeof(double) * L);
    double* tv = (double*)malloc(sizeof(double) * L);
    double* th = (double*)malloc(sizeof(double) * L);
    memcpy(x, x_init, sizeof(double) * L);
    double* w_l1 = wl;
    double* w_tv = wl + L;
    const int audit = lipschitz || trace != NULL;
    int nrows = 0;
    rc = OR_OK;

    for (int it = 0; it < c->inner_iters; ++it) {
        if (it == 0 || c->refresh == 0)
            or_compute_weights(n, x, c->eps, c->eps_prime, c->convex_mode, w_l1, w_tv);
        double lr = c->fixed_step;
        if (lipschitz) {
            double maxtv = 0.0;
            for (size_t m = 0; m < L; ++m)
                if (w_tv[m] > maxtv) maxtv = w_tv[m];
            lr = 1.0 / (2.0 * maxw + 2.0 * c->gamma + 12.0 * c->beta * maxtv / c->mu);
        }
        double before[7], after[7];
        if (audit) objective_with_weights(n, w, y, x, c, x_anchor, w_l1, w_tv, before);
        /* data_gradient re-checks the accumulator (regularizer.cpp:89); the
         * check was made above and the accumulator is const. */
        data_gradient_nocheck(n, w, y, x, g);
        if (c->beta > 0.0) or_smoothed_tv_gradient(n, x, c->mu, w_tv, tv);
        for (size_t m = 0; m < L; ++m) {
            double gs = 2.0 * g[m] + 2.0 * c->gamma * (x[m] - x_anchor[m]);
            if (c->beta > 0.0) gs += c->beta * tv[m];
            nx[m] = x[m] - lr * gs;
        }
        if (c->alpha > 0.0) {
            for (size_t m = 0; m < L; ++m) th[m] = lr * c->alpha * w_l1[m];
            or_prox_l1(n, nx, th, nx);
        }
        if (audit) {
            objective_with_weights(n, w, y, nx, c, x_anchor, w_l1, w_tv, after);
            if (lipschitz) {
                const double sb = surrogate(before);
                const double slack = 1e-9 * (fabs(sb) > 1.0 ? fabs(sb) : 1.0);
                if (surrogate(after) > sb + slack) {
                    rc = OR_ERR_STEP_DIVERGED;
                    break;
                }
            }
            if (trace) {
                memcpy(trace + 15 * (size_t)nrows, before, sizeof before);
                memcpy(trace + 15 * (size_t)nrows + 7, after, sizeof after);
                trace[15 * (size_t)nrows + 14] = lr;
                ++nrows;
            }
        }
        double* t = x;
        x = nx;
        nx = t;
    }
    if (rc == OR_OK) memcpy(x_out, x, sizeof(double) * L);
    if (rows) *rows = nrows;
    free(x);
    free(nx);
    free(wl);
    free(g);
    free(tv);
    free(th);
    return rc;
}

/* ---- setup (params.cpp:9-64) --------------------------------------------- */

int or_scale_data(int n, const double* w, const double* y, int finalized, double* s_y,
                  double* s_n) {
    if (!finalized) return OR_ERR_NON_HERMITIAN;
    const size_t L = vol(n);
    fftc_cplx* z = (fftc_cplx*)malloc(sizeof(fftc_cplx) * L);
    for (size_t m = 0; m < L; ++m) {
        if (w[m] > 0.0) {
            const double r = sqrt(w[m]);
            z[m].re = y[2 * m] / r;
            z[m].im = y[2 * m + 1] / r;
        } else {
            z[m].re = z[m].im = 0.0;
        }
    }
    fftc_3d(z, z, n, n, n, +1);
    const double inv = 1.0 / (double)L;
    /* ifft3's Hermitian guard (fourier.cpp:77-86, tol 1e-8) */
    double max_im = 0.0, max_abs = 0.0;
    for (size_t m = 0; m < L; ++m) {
        const double ai = fabs(z[m].im * inv);
        const double aa = sqrt(z[m].re * z[m].re + z[m].im * z[m].im) * inv;
        if (ai > max_im) max_im = ai;
        if (aa > max_abs) max_abs = aa;
    }
    if (max_abs > 0.0 && max_im / max_abs > 1e-8) {
        free(z);
        return OR_ERR_NON_HERMITIAN_INPUT;
    }
    double sq = 0.0, sw = 0.0;
    for (size_t m = 0; m < L; ++m) {
        const double v = z[m].re * inv;
        sq += v * v;
    }
    for (size_t m = 0; m < L; ++m) sw += w[m];
    free(z);
    *s_y = sqrt(sq / (double)L);
    *s_n = sw / (double)L;
    return OR_OK;
}

int or_derive_config(double s_y, double s_n, double eps, double eps_prime, double a, double b,
                     double g, or_reg_config* out) {
    if (s_y < 0.0 || s_n < 0.0) return OR_ERR_INVALID_ARGUMENT;
    if (!(eps > 0.0) || !(eps_prime > 0.0)) return OR_ERR_INVALID_ARGUMENT;
    if (a < 0.0 || b < 0.0 || g < 0.0) return OR_ERR_INVALID_ARGUMENT;
    if (s_y == 0.0 && (a > 0.0 || b > 0.0)) return OR_ERR_NON_POSITIVE_SCALE;
    memset(out, 0, sizeof *out);
    out->alpha = a * s_y * eps;
    out->beta = b * s_y * eps_prime;
    out->gamma = g * s_n;
    out->eps = eps;
    out->eps_prime = eps_prime;
    out->mu = 0.01 * eps_prime;
    out->inner_iters = 24;
    return or_validate_reg_config(out);
}
