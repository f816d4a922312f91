/* Minimal FFTW3 API shim — TEST INFRASTRUCTURE (oracle only).
 *
 * libfftw3 is not installed in this image. The reference's fourier.cpp uses
 * exactly four FFTW entry points (/root/reference/proj/src/fourier.cpp:22-29,
 * 37-44): fftw_plan_dft_3d, fftw_plan_dft_2d, fftw_execute and
 * fftw_destroy_plan, with FFTW_FORWARD/FFTW_BACKWARD and FFTW_ESTIMATE.
 * This header declares those with FFTW's published semantics (unnormalised,
 * row-major, last dimension fastest, forward sign -1) and routes them to the
 * oracle's own mixed-radix FFT (oracle/fftc.c). The shim is pinned by the
 * reference's own FFT known-answer tests (test_grid_fourier.cpp:29-121),
 * which oracle/Makefile runs.
 */
#ifndef CM_FFTW3_SHIM_H
#define CM_FFTW3_SHIM_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double fftw_complex[2];
typedef struct fftw_plan_s* fftw_plan;

#define FFTW_FORWARD (-1)
#define FFTW_BACKWARD (+1)
#define FFTW_MEASURE (0U)
#define FFTW_ESTIMATE (1U << 6)

fftw_plan fftw_plan_dft_3d(int n0, int n1, int n2, fftw_complex* in, fftw_complex* out,
                           int sign, unsigned flags);
fftw_plan fftw_plan_dft_2d(int n0, int n1, fftw_complex* in, fftw_complex* out, int sign,
                           unsigned flags);
void fftw_execute(const fftw_plan plan);
void fftw_destroy_plan(fftw_plan plan);

#ifdef __cplusplus
}
#endif
#endif
