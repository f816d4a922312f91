/* fftc — double-precision complex FFT used ONLY by the test oracle.
 *
 * TEST INFRASTRUCTURE. Nothing in the product path links this file: it is
 * the FFT underneath (a) the oracle's restatement of the reference solver
 * (oracle/cm_oracle.c) and (b) the FFTW3-API shim (oracle/fftw_shim/) that
 * lets the unmodified reference sources build without libfftw3.
 *
 * Convention follows /root/reference/proj/include/cryomap/fourier.hpp:6-9:
 * forward sums are unnormalised with exp(-2 pi i ...), the backward sum uses
 * exp(+2 pi i ...) and is also unnormalised here (the caller scales, exactly
 * as FFTW leaves scaling to the caller, fourier.cpp:72-73).
 *
 * Any length n >= 1 is supported: radix 4/2/3/5 Stockham stages plus a
 * generic odd-prime stage.
 */
#ifndef CM_ORACLE_FFTC_H
#define CM_ORACLE_FFTC_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { double re, im; } fftc_cplx;

/* Batched 1D transform of `batch` interleaved sequences of length n laid out
 * [n][batch] (element e of sequence b at data[e*batch + b]). sign = -1
 * forward, +1 backward. In place. */
void fftc_1d_batched(fftc_cplx* data, int n, int batch, int sign);

/* 3D transform of a row-major n0 x n1 x n2 array (n2 fastest), unnormalised.
 * in may equal out. */
void fftc_3d(const fftc_cplx* in, fftc_cplx* out, int n0, int n1, int n2, int sign);

/* 2D transform of a row-major n0 x n1 array (n1 fastest). */
void fftc_2d(const fftc_cplx* in, fftc_cplx* out, int n0, int n1, int sign);

#ifdef __cplusplus
}
#endif
#endif
