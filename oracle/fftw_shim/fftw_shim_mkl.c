/* FFTW3 API shim over oneMKL DFTI — TEST INFRASTRUCTURE (oracle only).
 *
 * Same contract as fftw_shim.c (see fftw3.h): the four FFTW entry points the
 * reference uses (/root/reference/proj/src/fourier.cpp:22-29, 37-44), FFTW's
 * published semantics (unnormalised both ways, row-major, last dimension
 * fastest, FFTW_FORWARD = -1 -> exp(-2 pi i ...)), a plan made and destroyed per
 * call like the reference's FFTW_ESTIMATE plans.
 *
 * Backend: oneMKL's DFTI, which the PyTorch wheel of this image links into
 * libtorch_cpu.so and exports (DftiCreateDescriptor_d_md, DftiSetValue,
 * DftiCommitDescriptor, DftiComputeForward/Backward, DftiFreeDescriptor).
 * mkl_dfti.h is not shipped, so the few enum values used are spelled out
 * below (oneMKL's published values; the shim is pinned by the reference's FFT
 * known-answer tests, test_grid_fourier.cpp:29-121, run by `make check`).
 *
 * Threads: DFTI_THREAD_LIMIT = $CM_REF_FFT_THREADS (default 1: the reference
 * never calls fftw_init_threads, so its FFTW transforms are single-threaded).
 * This replaces oracle/fftc.c as the CPU baseline's FFT (SURVEY §8(c)(1):
 * a tuned library FFT, not a home-made one, so the reference timing is fair).
 */
#include "fftw3.h"

#include <stdio.h>
#include <stdlib.h>

typedef void* dfti_handle;
long DftiCreateDescriptor_d_md(dfti_handle*, int domain, long dim, long* lengths);
long DftiSetValue(dfti_handle, int param, ...);
long DftiCommitDescriptor(dfti_handle);
long DftiComputeForward(dfti_handle, void*, ...);
long DftiComputeBackward(dfti_handle, void*, ...);
long DftiFreeDescriptor(dfti_handle*);
char* DftiErrorMessage(long);

enum {
    K_DFTI_PLACEMENT = 11,
    K_DFTI_THREAD_LIMIT = 27,
    K_DFTI_COMPLEX = 32,
    K_DFTI_INPLACE = 43,
    K_DFTI_NOT_INPLACE = 44,
};

struct fftw_plan_s {
    dfti_handle h;
    fftw_complex* in;
    fftw_complex* out;
    int sign;
};

static void check(long st, const char* what) {
    if (st != 0) {
        fprintf(stderr, "fftw_shim_mkl: %s failed: %s\n", what, DftiErrorMessage(st));
        abort();
    }
}

static int shim_threads(void) {
    const char* s = getenv("CM_REF_FFT_THREADS");
    int t = s ? atoi(s) : 1;
    return t > 0 ? t : 1;
}

static fftw_plan make_plan(int rank, long* lengths, fftw_complex* in, fftw_complex* out,
                           int sign) {
    fftw_plan p = (fftw_plan)malloc(sizeof(*p));
    p->in = in;
    p->out = out;
    p->sign = sign;
    check(DftiCreateDescriptor_d_md(&p->h, K_DFTI_COMPLEX, rank, lengths), "create");
    check(DftiSetValue(p->h, K_DFTI_PLACEMENT, in == out ? K_DFTI_INPLACE : K_DFTI_NOT_INPLACE),
          "placement");
    check(DftiSetValue(p->h, K_DFTI_THREAD_LIMIT, shim_threads()), "thread limit");
    check(DftiCommitDescriptor(p->h), "commit");
    return p;
}

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags) {
    (void)flags;
    long L[3] = {n0, n1, n2};
    return make_plan(3, L, in, out, sign);
}

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)flags;
    long L[2] = {n0, n1};
    return make_plan(2, L, in, out, sign);
}

void fftw_execute(const fftw_plan p) {
    if (p->in == p->out)
        check(p->sign == FFTW_FORWARD ? DftiComputeForward(p->h, p->in)
                                      : DftiComputeBackward(p->h, p->in),
              "compute");
    else
        check(p->sign == FFTW_FORWARD ? DftiComputeForward(p->h, p->in, p->out)
                                      : DftiComputeBackward(p->h, p->in, p->out),
              "compute");
}

void fftw_destroy_plan(fftw_plan p) {
    DftiFreeDescriptor(&p->h);
    free(p);
}
