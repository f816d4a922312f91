/* fftc — see fftc.h. TEST INFRASTRUCTURE ONLY (oracle + FFTW-API shim). */
#include "fftc.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define FFTC_MAXF 64

typedef struct {
    int n;
    int nf;
    int radix[FFTC_MAXF];
    fftc_cplx* tw; /* tw[t] = exp(sign * 2 pi i t / n), t in [0, n) */
} fftc_plan;

static void plan_make(fftc_plan* p, int n, int sign) {
    p->n = n;
    p->nf = 0;
    int m = n;
    while (m % 4 == 0) { p->radix[p->nf++] = 4; m /= 4; }
    while (m % 2 == 0) { p->radix[p->nf++] = 2; m /= 2; }
    while (m % 3 == 0) { p->radix[p->nf++] = 3; m /= 3; }
    while (m % 5 == 0) { p->radix[p->nf++] = 5; m /= 5; }
    for (int f = 7; m > 1; f += 2)
        while (m % f == 0) { p->radix[p->nf++] = f; m /= f; }
    p->tw = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)(n > 0 ? n : 1));
    const double two_pi = 6.283185307179586476925286766559;
    for (int t = 0; t < n; ++t) {
        const double a = sign * two_pi * (double)t / (double)n;
        p->tw[t].re = cos(a);
        p->tw[t].im = sin(a);
    }
}

static void plan_free(fftc_plan* p) { free(p->tw); }

/* One Stockham stage: src/dst are [n][B]. */
static void stage(const fftc_plan* p, int R, int Ns, const fftc_cplx* src, fftc_cplx* dst,
                  int B, int sign) {
    const int n = p->n;
    const int nR = n / R;
    const int tstep = n / (Ns * R);
    fftc_cplx v[FFTC_MAXF > 32 ? 32 : FFTC_MAXF];
    fftc_cplx* vb = NULL;
    if (R > 32) vb = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)R);
    fftc_cplx* vv = vb ? vb : v;
    const double s = (double)sign;
    for (int j = 0; j < nR; ++j) {
        const int k = j % Ns;
        const int idxD = (j / Ns) * Ns * R + k;
        for (int b = 0; b < B; ++b) {
            for (int r = 0; r < R; ++r) {
                fftc_cplx x = src[(size_t)(j + r * nR) * B + b];
                if (k != 0 && r != 0) {
                    const fftc_cplx w = p->tw[(r * k * tstep) % n];
                    const double re = x.re * w.re - x.im * w.im;
                    const double im = x.re * w.im + x.im * w.re;
                    x.re = re;
                    x.im = im;
                }
                vv[r] = x;
            }
            if (R == 2) {
                fftc_cplx a = vv[0], c = vv[1];
                vv[0].re = a.re + c.re; vv[0].im = a.im + c.im;
                vv[1].re = a.re - c.re; vv[1].im = a.im - c.im;
            } else if (R == 4) {
                fftc_cplx a0 = vv[0], a1 = vv[1], a2 = vv[2], a3 = vv[3];
                double t0r = a0.re + a2.re, t0i = a0.im + a2.im;
                double t1r = a0.re - a2.re, t1i = a0.im - a2.im;
                double t2r = a1.re + a3.re, t2i = a1.im + a3.im;
                double t3r = a1.re - a3.re, t3i = a1.im - a3.im;
                /* multiply t3 by sign*i */
                double u3r = -s * t3i, u3i = s * t3r;
                vv[0].re = t0r + t2r; vv[0].im = t0i + t2i;
                vv[2].re = t0r - t2r; vv[2].im = t0i - t2i;
                vv[1].re = t1r + u3r; vv[1].im = t1i + u3i;
                vv[3].re = t1r - u3r; vv[3].im = t1i - u3i;
            } else if (R == 3) {
                const double c1 = -0.5, s1 = s * 0.86602540378443864676372317075294;
                fftc_cplx a0 = vv[0], a1 = vv[1], a2 = vv[2];
                double sr = a1.re + a2.re, si = a1.im + a2.im;
                double dr = a1.re - a2.re, di = a1.im - a2.im;
                vv[0].re = a0.re + sr;
                vv[0].im = a0.im + si;
                double mr = a0.re + c1 * sr, mi = a0.im + c1 * si;
                /* (dr + i di) * (i s1) = -s1 di + i s1 dr */
                vv[1].re = mr - s1 * di; vv[1].im = mi + s1 * dr;
                vv[2].re = mr + s1 * di; vv[2].im = mi - s1 * dr;
            } else {
                /* generic DFT of length R */
                fftc_cplx out[32];
                fftc_cplx* o = out;
                fftc_cplx* ob = NULL;
                if (R > 32) { ob = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)R); o = ob; }
                const int step = n / R;
                for (int q = 0; q < R; ++q) {
                    double re = 0.0, im = 0.0;
                    for (int r = 0; r < R; ++r) {
                        const fftc_cplx w = p->tw[((q * r) % R) * step];
                        re += vv[r].re * w.re - vv[r].im * w.im;
                        im += vv[r].re * w.im + vv[r].im * w.re;
                    }
                    o[q].re = re;
                    o[q].im = im;
                }
                for (int q = 0; q < R; ++q) vv[q] = o[q];
                free(ob);
            }
            for (int r = 0; r < R; ++r) dst[(size_t)(idxD + r * Ns) * B + b] = vv[r];
        }
    }
    free(vb);
}

/* data [n][B] in place; work is a scratch of the same size. */
static void run_plan(const fftc_plan* p, fftc_cplx* data, fftc_cplx* work, int B, int sign) {
    fftc_cplx* src = data;
    fftc_cplx* dst = work;
    int Ns = 1;
    for (int f = 0; f < p->nf; ++f) {
        const int R = p->radix[f];
        stage(p, R, Ns, src, dst, B, sign);
        Ns *= R;
        fftc_cplx* t = src;
        src = dst;
        dst = t;
    }
    if (src != data) memcpy(data, src, sizeof(fftc_cplx) * (size_t)p->n * (size_t)B);
}

void fftc_1d_batched(fftc_cplx* data, int n, int batch, int sign) {
    if (n <= 1 || batch <= 0) return;
    fftc_plan p;
    plan_make(&p, n, sign);
    fftc_cplx* work = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)n * (size_t)batch);
    run_plan(&p, data, work, batch, sign);
    free(work);
    plan_free(&p);
}

/* Transform `count` sequences of length n: sequence q has element e at
 * a[q_base(q) + e*es]. Sequences are processed CH at a time through a
 * contiguous [n][CH] buffer. */
#define FFTC_CH 16

static void axis_pass(fftc_cplx* a, int n, size_t es, size_t count, size_t inner,
                      size_t outer_stride, int sign) {
    /* sequences are indexed (o, c) with base = o*outer_stride + c for
     * c in [0, inner); count = number of o values. */
    if (n <= 1) return;
    fftc_plan p;
    plan_make(&p, n, sign);
    fftc_cplx* buf = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)n * FFTC_CH);
    fftc_cplx* work = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)n * FFTC_CH);
    for (size_t o = 0; o < count; ++o) {
        for (size_t c0 = 0; c0 < inner; c0 += FFTC_CH) {
            const int B = (int)((inner - c0) < FFTC_CH ? (inner - c0) : FFTC_CH);
            fftc_cplx* base = a + o * outer_stride + c0;
            for (int e = 0; e < n; ++e)
                for (int b = 0; b < B; ++b) buf[(size_t)e * B + b] = base[(size_t)e * es + b];
            run_plan(&p, buf, work, B, sign);
            for (int e = 0; e < n; ++e)
                for (int b = 0; b < B; ++b) base[(size_t)e * es + b] = buf[(size_t)e * B + b];
        }
    }
    free(buf);
    free(work);
    plan_free(&p);
}

/* contiguous lines: gather CH lines transposed into [n][CH] */
static void line_pass(fftc_cplx* a, int n, size_t lines, int sign) {
    if (n <= 1) return;
    fftc_plan p;
    plan_make(&p, n, sign);
    fftc_cplx* buf = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)n * FFTC_CH);
    fftc_cplx* work = (fftc_cplx*)malloc(sizeof(fftc_cplx) * (size_t)n * FFTC_CH);
    for (size_t l0 = 0; l0 < lines; l0 += FFTC_CH) {
        const int B = (int)((lines - l0) < FFTC_CH ? (lines - l0) : FFTC_CH);
        fftc_cplx* base = a + l0 * (size_t)n;
        for (int b = 0; b < B; ++b)
            for (int e = 0; e < n; ++e) buf[(size_t)e * B + b] = base[(size_t)b * n + e];
        run_plan(&p, buf, work, B, sign);
        for (int b = 0; b < B; ++b)
            for (int e = 0; e < n; ++e) base[(size_t)b * n + e] = buf[(size_t)e * B + b];
    }
    free(buf);
    free(work);
    plan_free(&p);
}

void fftc_3d(const fftc_cplx* in, fftc_cplx* out, int n0, int n1, int n2, int sign) {
    const size_t total = (size_t)n0 * n1 * n2;
    if (in != out) memcpy(out, in, sizeof(fftc_cplx) * total);
    /* axis 2: contiguous lines */
    line_pass(out, n2, (size_t)n0 * n1, sign);
    /* axis 1: for each plane o, columns c in [0,n2), element stride n2 */
    axis_pass(out, n1, (size_t)n2, (size_t)n0, (size_t)n2, (size_t)n1 * n2, sign);
    /* axis 0: one "plane" of n1*n2 columns, element stride n1*n2 */
    axis_pass(out, n0, (size_t)n1 * n2, 1, (size_t)n1 * n2, 0, sign);
}

void fftc_2d(const fftc_cplx* in, fftc_cplx* out, int n0, int n1, int sign) {
    const size_t total = (size_t)n0 * n1;
    if (in != out) memcpy(out, in, sizeof(fftc_cplx) * total);
    line_pass(out, n1, (size_t)n0, sign);
    axis_pass(out, n0, (size_t)n1, 1, (size_t)n1, 0, sign);
}
