/* FFTW3 API shim over oracle/fftc.c — TEST INFRASTRUCTURE (oracle only).
 * See fftw3.h for the contract. */
#include "fftw3.h"

#include <stdlib.h>

#include "../fftc.h"

struct fftw_plan_s {
    int rank;
    int n0, n1, n2;
    fftw_complex* in;
    fftw_complex* out;
    int sign;
};

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags) {
    (void)flags;
    fftw_plan p = (fftw_plan)malloc(sizeof(*p));
    p->rank = 3;
    p->n0 = n0;
    p->n1 = n1;
    p->n2 = n2;
    p->in = in;
    p->out = out;
    p->sign = sign;
    return p;
}

fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags) {
    (void)flags;
    fftw_plan p = (fftw_plan)malloc(sizeof(*p));
    p->rank = 2;
    p->n0 = n0;
    p->n1 = n1;
    p->n2 = 1;
    p->in = in;
    p->out = out;
    p->sign = sign;
    return p;
}

void fftw_execute(const fftw_plan p) {
    if (p->rank == 3)
        fftc_3d((const fftc_cplx*)p->in, (fftc_cplx*)p->out, p->n0, p->n1, p->n2, p->sign);
    else
        fftc_2d((const fftc_cplx*)p->in, (fftc_cplx*)p->out, p->n0, p->n1, p->sign);
}

void fftw_destroy_plan(fftw_plan p) { free(p); }
