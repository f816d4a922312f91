// E-step on the device (reference: e_step,
// estep.cpp:64-270, with sample_slice slice.cpp:24-45).
//
// Posterior over (pose, shift) candidates per particle, proportional to
// exp(-R/2) with the whitened residual
//   R = A + b - 2 Re sum_j (w ctf X_j) conj(S_j) ph_s,j,
//   A = sum_j w |X_j|^2,  b = sum_j w ctf^2 |S_j|^2,
// the reference's exact-safe pose pruning (lower bound LB = A + b - 2 sum_j
// w |ctf| |X_j| |S_j| against the best zero-shift residual U plus
// 2 ln(1 / prune_floor)), a max-subtracted softmax over the surviving
// candidates, then the prune_floor cut and renormalisation.
//
// Mapping: slices S[pose][j] are gathered once (one thread per pose and
// component: the 27 / 8 kernel taps of the rotated frequency, 24 MB at 128^2 x
// 100 poses -- L2-resident for the sweeps); the per-particle tables
// (w ctf X, w ctf^2, w |ctf| |X|) once; then one CTA per (particle, pose)
// reduces over the components, particle-major so a particle's table and all
// slices stay in L2 while its poses are swept. Pass 2 evaluates all shifts of
// two poses at a time from one read of the particle's terms and the phases.
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../include/cm_api.h"
#include "backproject.cuh"
#include "cm_common.cuh"

namespace cm {

struct EsDev {
    const double2* V;       // FourierVolume [n^3] (storage indices)
    const double2* img;     // [npart][n*n]
    const double* ip;       // [npart][6]
    const double* mats;     // [npose][9]
    const int2* comps;      // [ncomp]
    const double* invsig;   // [ncomp]
    double* phr;            // [nshift][ncomp]
    double* phi;
    double2* slice;         // [npose][ncomp]
    double *p1r, *p1i, *p2, *pab;  // [npart][ncomp]
    double *A, *R0, *LB, *U;
    double* res;            // [npart][npose * nshift]
    int n, ncomp, npose, nshift, npart;
    double slack, floor_, bandwidth;
    const int* sidx;        // [nsh2] the shifts pass 2 evaluates (all but the zero shift)
    int nsh2, zsh;          // zsh: index of the zero shift (-1: none); its residual is R0
};

constexpr int ES_NT = 256;

template <int NV>
__device__ __forceinline__ void es_block_sum(double (&v)[NV], double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < NV; ++q)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_xor_sync(0xffffffffu, v[q], o);
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int q = 0; q < NV; ++q) red[w * NV + q] = v[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NV; ++q) {
        double s = 0.0;
        for (int k = 0; k < ES_NT / 32; ++k) s += red[k * NV + q];
        v[q] = s;
    }
}

__device__ __forceinline__ double es_block_min(double v, double* red) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[w] = v;
    __syncthreads();
    double s = red[0];
    for (int k = 1; k < ES_NT / 32; ++k) s = fmin(s, red[k]);
    return s;
}

// sample_slice (slice.cpp:24-45): kernel-weighted normalised interpolation
template <int KIND>
__global__ void es_slice_kernel(EsDev p) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)p.npose * p.ncomp) return;
    const int pose = (int)(t / p.ncomp), j = (int)(t % p.ncomp);
    const int n = p.n, lo = -n / 2, hi = n / 2 - 1;
    const double* R = p.mats + 9 * (size_t)pose;
    const int k = p.comps[j].x, l = p.comps[j].y;
    double nj[3];
#pragma unroll
    for (int a = 0; a < 3; ++a)  // as in backproject.cuh (the reference's as-built order)
        nj[a] = __dadd_rn(__fma_rn(R[3 * a], (double)k, __dmul_rn(R[3 * a + 1], (double)l)),
                          __dmul_rn(R[3 * a + 2], 0.0));
    double ar = 0.0, ai = 0.0, ws = 0.0;
    auto tap = [&](int px, int py, int pz, double w) {
        if (px < lo || px > hi || py < lo || py > hi || pz < lo || pz > hi) return;
        const double2 v = p.V[((size_t)bp_store(pz, n) * n + bp_store(py, n)) * n + bp_store(px, n)];
        ar += w * v.x;
        ai += w * v.y;
        ws += w;
    };
    if constexpr (KIND == 0) {
        int anc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) anc[a] = (int)llround(nj[a]);
        for (int dz = -1; dz <= 1; ++dz)
            for (int dy = -1; dy <= 1; ++dy)
                for (int dx = -1; dx <= 1; ++dx) {
                    const int q[3] = {anc[0] + dx, anc[1] + dy, anc[2] + dz};
                    double d2 = 0.0;
#pragma unroll
                    for (int a = 0; a < 3; ++a) {
                        const double d = nj[a] - (double)q[a];
                        d2 += d * d;
                    }
                    tap(q[0], q[1], q[2], exp(-d2 / p.bandwidth));
                }
    } else {
        int lo3[3];
        double fr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo3[a] = (int)floor(nj[a]);
            fr[a] = nj[a] - (double)lo3[a];
        }
        const int cz1 = fr[2] == 0.0 ? 0 : 1, cy1 = fr[1] == 0.0 ? 0 : 1, cx1 = fr[0] == 0.0 ? 0 : 1;
        for (int cz = 0; cz <= cz1; ++cz)
            for (int cy = 0; cy <= cy1; ++cy)
                for (int cx = 0; cx <= cx1; ++cx)
                    tap(lo3[0] + cx, lo3[1] + cy, lo3[2] + cz,
                        (cx ? fr[0] : 1.0 - fr[0]) * (cy ? fr[1] : 1.0 - fr[1]) *
                            (cz ? fr[2] : 1.0 - fr[2]));
    }
    p.slice[t] = ws > 0.0 ? make_double2(ar / ws, ai / ws) : make_double2(0.0, 0.0);
}

// shift phase tables (slice.cpp:47-50), [nshift][ncomp]
__global__ void es_phase_kernel(EsDev p, const int2* shifts) {
    const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (t >= (long long)p.nshift * p.ncomp) return;
    const int s = (int)(t / p.ncomp), j = (int)(t % p.ncomp);
    const int k = p.comps[j].x, l = p.comps[j].y;
    const double ph = -2.0 * 3.14159265358979323846 * ((double)k * shifts[s].x + (double)l * shifts[s].y) /
                      (double)p.n;
    double sn, cs;
    sincos(ph, &sn, &cs);
    p.phr[t] = cs;
    p.phi[t] = sn;
}

// per-particle tables (estep.cpp:167-186) and A by one CTA per particle
__global__ void __launch_bounds__(ES_NT) es_ptab_kernel(EsDev p) {
    __shared__ double red[ES_NT / 32];
    const int part = blockIdx.x, n = p.n;
    const double* ip = p.ip + 6 * (size_t)part;
    double a = 0.0;
    for (int j = threadIdx.x; j < p.ncomp; j += ES_NT) {
        const int k = p.comps[j].x, l = p.comps[j].y;
        const double s = __dsqrt_rn((double)(k * k + l * l)) / ((double)n * ip[5]);
        const double ctf = bp_ctf(ip, s);
        const double w = p.invsig[j];
        const double2 x = p.img[(size_t)part * n * n + (size_t)bp_store(l, n) * n + bp_store(k, n)];
        a += w * (x.x * x.x + x.y * x.y);
        const size_t o = (size_t)part * p.ncomp + j;
        const double wc = w * ctf;
        p.p1r[o] = wc * x.x;
        p.p1i[o] = wc * x.y;
        p.p2[o] = wc * ctf;
        p.pab[o] = w * fabs(ctf) * hypot(x.x, x.y);
    }
    double v[1] = {a};
    es_block_sum<1>(v, red);
    if (threadIdx.x == 0) p.A[part] = v[0];
}

// pass 1 (estep.cpp:189-208): zero-shift residual R0 and the bound LB
__global__ void __launch_bounds__(ES_NT) es_pass1_kernel(EsDev p) {
    __shared__ double red[3 * ES_NT / 32];
    const int part = blockIdx.x / p.npose, pose = blockIdx.x % p.npose;
    const double* p1r = p.p1r + (size_t)part * p.ncomp;
    const double* p1i = p.p1i + (size_t)part * p.ncomp;
    const double* p2 = p.p2 + (size_t)part * p.ncomp;
    const double* pa = p.pab + (size_t)part * p.ncomp;
    const double2* S = p.slice + (size_t)pose * p.ncomp;
    double v[3] = {0.0, 0.0, 0.0};  // b, cross, absum
    for (int j = threadIdx.x; j < p.ncomp; j += ES_NT) {
        const double2 s = S[j];
        const double t1 = s.x * s.x + s.y * s.y;
        v[0] += p2[j] * t1;
        v[1] += p1r[j] * s.x + p1i[j] * s.y;
        v[2] += pa[j] * sqrt(t1);
    }
    es_block_sum<3>(v, red);
    if (threadIdx.x == 0) {
        const double A = p.A[part];
        p.R0[blockIdx.x] = A + v[0] - 2.0 * v[1];
        p.LB[blockIdx.x] = A + v[0] - 2.0 * v[2];
    }
}

// U: best zero-shift residual per particle (estep.cpp:210-215)
__global__ void __launch_bounds__(ES_NT) es_min_kernel(EsDev p) {
    __shared__ double red[ES_NT / 32];
    const int part = blockIdx.x;
    double m = INFINITY;
    for (int q = threadIdx.x; q < p.npose; q += ES_NT) m = fmin(m, p.R0[(size_t)part * p.npose + q]);
    m = es_block_min(m, red);
    if (threadIdx.x == 0) p.U[part] = m;
}

// pass 2 (estep.cpp:217-249): every shift of each surviving (particle, pose).
// One CTA per particle and group of ES_PG poses: the particle's terms and the
// shift-phase tables are read once per group instead of once per pose; the
// zero shift is pass 1's R0 (13 shifts -> 3 batches of 4, not 4); PG = 2,
// SB = 4 keeps it at 2 CTAs / SM without spills (PG = 4 needs 250 registers).
constexpr int ES_PG = 2, ES_SB = 4;
__global__ void __launch_bounds__(ES_NT, 2) es_pass2_kernel(EsDev p) {
    constexpr int PG = ES_PG, SB = ES_SB, NV = PG * SB + PG;
    __shared__ double red[NV * ES_NT / 32];
    const int ngrp = (p.npose + PG - 1) / PG;
    const int part = blockIdx.x / ngrp, pose0 = (blockIdx.x % ngrp) * PG;
    const double U = p.U[part] + p.slack;
    bool alive[PG];
    bool any = false;
#pragma unroll
    for (int g = 0; g < PG; ++g) {
        const int pose = pose0 + g;
        alive[g] = pose < p.npose && !(p.LB[(size_t)part * p.npose + pose] > U);
        any |= alive[g];
        if (pose < p.npose && !alive[g]) {  // pruned pose: no candidates
            double* out = p.res + ((size_t)part * p.npose + pose) * p.nshift;
            for (int s = threadIdx.x; s < p.nshift; s += ES_NT) out[s] = INFINITY;
        }
    }
    if (!any) return;
    const double* p1r = p.p1r + (size_t)part * p.ncomp;
    const double* p1i = p.p1i + (size_t)part * p.ncomp;
    const double* p2 = p.p2 + (size_t)part * p.ncomp;
    if (p.zsh >= 0 && threadIdx.x == 0)  // the zero shift's residual is pass 1's R0
#pragma unroll
        for (int g = 0; g < PG; ++g)
            if (alive[g])
                p.res[((size_t)part * p.npose + pose0 + g) * p.nshift + p.zsh] =
                    p.R0[(size_t)part * p.npose + pose0 + g];
    double base[PG];
    for (int s0 = 0; s0 < p.nsh2; s0 += SB) {
        double v[NV];
#pragma unroll
        for (int q = 0; q < NV; ++q) v[q] = 0.0;
        for (int j = threadIdx.x; j < p.ncomp; j += ES_NT) {
            const double ar = p1r[j], ai = p1i[j], a2 = p2[j];
            double phr[SB], phi[SB];
#pragma unroll
            for (int q = 0; q < SB; ++q) {
                const bool ok = s0 + q < p.nsh2;
                const size_t o = (size_t)(ok ? p.sidx[s0 + q] : 0) * p.ncomp + j;
                phr[q] = ok ? p.phr[o] : 0.0;
                phi[q] = ok ? p.phi[o] : 0.0;
            }
#pragma unroll
            for (int g = 0; g < PG; ++g) {
                if (!alive[g]) continue;
                const double2 sv = p.slice[(size_t)(pose0 + g) * p.ncomp + j];
                if (s0 == 0) v[PG * SB + g] += a2 * (sv.x * sv.x + sv.y * sv.y);
                const double cr = ar * sv.x + ai * sv.y;
                const double ci = ai * sv.x - ar * sv.y;
#pragma unroll
                for (int q = 0; q < SB; ++q) v[g * SB + q] += cr * phr[q] + ci * phi[q];
            }
        }
        es_block_sum<NV>(v, red);
#pragma unroll
        for (int g = 0; g < PG; ++g) {
            if (s0 == 0) base[g] = p.A[part] + v[PG * SB + g];
            if (threadIdx.x == 0 && alive[g]) {
                double* out = p.res + ((size_t)part * p.npose + pose0 + g) * p.nshift;
                for (int q = 0; q < SB && s0 + q < p.nsh2; ++q) out[p.sidx[s0 + q]] = base[g] - 2.0 * v[g * SB + q];
            }
        }
    }
}

// softmax, prune, renormalise (estep.cpp:251-268): dense posterior row
__global__ void __launch_bounds__(ES_NT) es_softmax_kernel(EsDev p, double* post) {
    __shared__ double red[ES_NT / 32];
    const int part = blockIdx.x;
    const int nc = p.npose * p.nshift;
    const double* r = p.res + (size_t)part * nc;
    double* o = post + (size_t)part * nc;
    double m = INFINITY;
    for (int c = threadIdx.x; c < nc; c += ES_NT) m = fmin(m, r[c]);
    const double rmin = es_block_min(m, red);
    double v[1] = {0.0};
    for (int c = threadIdx.x; c < nc; c += ES_NT)
        if (r[c] < INFINITY) v[0] += exp(-(r[c] - rmin) / 2.0);
    es_block_sum<1>(v, red);
    const double z = v[0];
    double kv[1] = {0.0};
    for (int c = threadIdx.x; c < nc; c += ES_NT) {
        double w = 0.0;
        if (r[c] < INFINITY) {
            w = exp(-(r[c] - rmin) / 2.0) / z;
            if (!(w >= p.floor_)) w = 0.0;
        }
        o[c] = w;
        kv[0] += w;
    }
    es_block_sum<1>(kv, red);
    const double kept = kv[0];
    // every candidate below prune_floor: the reference's row is empty
    // (estep.cpp:257-263 pushes no entry), not 0/0
    for (int c = threadIdx.x; c < nc; c += ES_NT) o[c] = kept > 0.0 ? o[c] / kept : 0.0;
}

// nonzero entries per posterior row (one CTA per particle)
__global__ void __launch_bounds__(ES_NT) es_count_kernel(const double* post, int nc, int* cnt) {
    __shared__ double red[ES_NT / 32];
    const double* o = post + (size_t)blockIdx.x * nc;
    double v[1] = {0.0};
    for (int c = threadIdx.x; c < nc; c += ES_NT) v[0] += o[c] != 0.0 ? 1.0 : 0.0;
    es_block_sum<1>(v, red);
    if (threadIdx.x == 0) cnt[blockIdx.x] = (int)v[0];
}

// PosteriorRow entries (estep.hpp:30-34) in ascending candidate order, as the
// reference pushes them (estep.cpp:257-263): block-wide prefix sums per chunk
__global__ void __launch_bounds__(ES_NT) es_compact_kernel(const double* post, int nc,
                                                           const long long* off, int* cand,
                                                           double* wout) {
    __shared__ int wsum[ES_NT / 32];
    __shared__ int base_s;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const double* o = post + (size_t)blockIdx.x * nc;
    long long base = off[blockIdx.x];
    for (int c0 = 0; c0 < nc; c0 += ES_NT) {
        const int c = c0 + threadIdx.x;
        const double v = c < nc ? o[c] : 0.0;
        const int f = v != 0.0 ? 1 : 0;
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        const int pre = __popc(bal & ((1u << lane) - 1u));
        if (lane == 0) wsum[w] = __popc(bal);
        __syncthreads();
        int wpre = 0, tot = 0;
        for (int k = 0; k < ES_NT / 32; ++k) {
            wpre += k < w ? wsum[k] : 0;
            tot += wsum[k];
        }
        if (f) {
            cand[base + wpre + pre] = c;
            wout[base + wpre + pre] = v;
        }
        if (threadIdx.x == 0) base_s = tot;
        __syncthreads();
        base += base_s;
        __syncthreads();
    }
}

// Where a batch's posterior rows go: the dense host matrix [np][nc], or the
// sparse PosteriorRow lists (row_ptr [np+1], candidate / weight of capacity cap)
struct EsSink {
    double* dense = nullptr;
    long long* row_ptr = nullptr;
    int* cand = nullptr;
    double* weight = nullptr;
    long long cap = 0;
    long long nnz = 0;      // entries so far (required count when over capacity)
    bool overflow = false;
};

// Host side. V: device FourierVolume (host upload or the resident spectrum).
// Particles are processed in batches sized to CM_ESTEP_BATCH_BYTES of device
// scratch (default 1 GiB): the per-particle tables, residuals and posterior
// rows of one batch; the slices and shift phases are built once per call.
inline int estep_run(int n, const cm_estep_input* in, const double* V_host, const double* V_dev,
                     EsSink& sink, cudaStream_t st, const ParticleDev* resident = nullptr) {
    if (in->n_poses <= 0 || in->n_shifts <= 0)
        return fail(CM_ERR_INVALID_ARGUMENT, "e_step: empty orientation grid");
    if (in->kernel_kind != 0 && in->kernel_kind != 1)
        return fail(CM_ERR_INVALID_ARGUMENT, "e_step: unknown kernel kind");
    if (in->kernel_kind == 0 && !(in->bandwidth > 0.0))
        return fail(CM_ERR_INVALID_ARGUMENT, "gaussian kernel bandwidth must be positive");
    if (in->n_images < 0 || !in->poses || !in->shifts || in->n_sigma2 < 1 || !in->sigma2)
        return fail(CM_ERR_INVALID_ARGUMENT, "e_step: missing input array");
    bool host_images = true;
    if (in->n_images > 0) CKS(particles_of(in->n_images, in->images, in->image_params, resident, &host_images));
    if (!(in->prune_floor > 0.0)) return fail(CM_ERR_INVALID_ARGUMENT, "e_step: prune_floor must be positive");
    bool zero_shift = false;
    for (int s = 0; s < in->n_shifts; ++s)
        zero_shift |= in->shifts[2 * s] == 0 && in->shifts[2 * s + 1] == 0;
    if (!zero_shift) return fail(CM_ERR_INVALID_ARGUMENT, "e_step: orientation grid lacks the zero shift");
    if (sink.row_ptr) sink.row_ptr[0] = 0;
    if (in->n_images == 0) return CM_OK;
    // build_comp_tables (estep.cpp:26-40) with effective_cutoff (:14-17)
    const double nyq = double(n / 2);
    const double cutoff = in->radius_cutoff < 0.0 ? nyq : std::min(in->radius_cutoff, nyq);
    std::vector<int2> comps;
    std::vector<double> invsig;
    for (int b = 0; b < n; ++b)
        for (int a = 0; a < n; ++a) {
            const int k = a < n / 2 ? a : a - n, l = b < n / 2 ? b : b - n;
            const long r = std::lround(std::hypot(double(k), double(l)));
            if (r > std::lround(cutoff)) continue;
            comps.push_back(make_int2(k, l));
            invsig.push_back(1.0 / in->sigma2[std::min<long>(r, in->n_sigma2 - 1)]);
        }
    std::vector<double> mats(9 * (size_t)in->n_poses);
    for (int q = 0; q < in->n_poses; ++q) bp_rotation(in->poses + 3 * (size_t)q, mats.data() + 9 * (size_t)q);
    const int ncomp = (int)comps.size(), np = in->n_images, npose = in->n_poses, ns = in->n_shifts;
    const size_t L = (size_t)n * n * n, nc = (size_t)npose * ns;

    // batch size: device bytes per particle of the batch-local arrays
    size_t budget = size_t(1) << 30;
    if (const char* e = std::getenv("CM_ESTEP_BATCH_BYTES")) budget = std::max<size_t>(1, std::strtoull(e, nullptr, 10));
    const size_t per_part = 8 * (4 * (size_t)ncomp + 2 + 2 * (size_t)npose + 2 * nc) +
                            (host_images ? 16 * (size_t)n * n + 48 : 0) + 16;
    const int nb = (int)std::max<size_t>(1, std::min<size_t>((size_t)np, budget / per_part));

    BpBuffers B;
    double2* Vd = nullptr;
    double *dm = nullptr, *isg = nullptr, *phr = nullptr, *phi = nullptr;
    int2 *cmp = nullptr, *shf = nullptr;
    double2* slice = nullptr;
    if (V_host) CKS(B.put(&Vd, reinterpret_cast<const double2*>(V_host), L, st));
    CKS(B.put(&dm, mats.data(), mats.size(), st));
    CKS(B.put(&cmp, comps.data(), comps.size(), st));
    CKS(B.put(&isg, invsig.data(), invsig.size(), st));
    CKS(B.put(&shf, reinterpret_cast<const int2*>(in->shifts), (size_t)ns, st));
    CKS(B.put(&phr, (const double*)nullptr, (size_t)ns * ncomp, st));
    CKS(B.put(&phi, (const double*)nullptr, (size_t)ns * ncomp, st));
    CKS(B.put(&slice, (const double2*)nullptr, (size_t)npose * ncomp, st));
    // batch-local arrays
    double2* img_b = nullptr;
    double* ip_b = nullptr;
    if (host_images) {
        CKS(B.put(&img_b, (const double2*)nullptr, (size_t)nb * n * n, st));
        CKS(B.put(&ip_b, (const double*)nullptr, (size_t)nb * 6, st));
    }
    double *p1r = nullptr, *p1i = nullptr, *p2 = nullptr, *pab = nullptr, *A = nullptr, *R0 = nullptr,
           *LB = nullptr, *U = nullptr, *res = nullptr, *post = nullptr;
    for (double** q : {&p1r, &p1i, &p2, &pab}) CKS(B.put(q, (const double*)nullptr, (size_t)nb * ncomp, st));
    CKS(B.put(&A, (const double*)nullptr, (size_t)nb, st));
    CKS(B.put(&U, (const double*)nullptr, (size_t)nb, st));
    CKS(B.put(&R0, (const double*)nullptr, (size_t)nb * npose, st));
    CKS(B.put(&LB, (const double*)nullptr, (size_t)nb * npose, st));
    CKS(B.put(&res, (const double*)nullptr, (size_t)nb * nc, st));
    CKS(B.put(&post, (const double*)nullptr, (size_t)nb * nc, st));
    int* cnt = nullptr;
    long long* offd = nullptr;
    if (sink.row_ptr) {
        CKS(B.put(&cnt, (const int*)nullptr, (size_t)nb, st));
        CKS(B.put(&offd, (const long long*)nullptr, (size_t)nb, st));
    }
    EsDev p{V_host ? Vd : reinterpret_cast<const double2*>(V_dev), nullptr, nullptr, dm, cmp, isg, phr, phi,
            slice, p1r, p1i, p2, pab, A, R0, LB, U, res, n, ncomp, npose, ns, 0,
            2.0 * std::log(1.0 / in->prune_floor), in->prune_floor, in->bandwidth};
    // pass 2 skips the zero shift: its residual is pass 1's R0 (the same sums)
    std::vector<int> sidx;
    int zsh = -1;
    for (int q = 0; q < ns; ++q) {
        if (zsh < 0 && in->shifts[2 * q] == 0 && in->shifts[2 * q + 1] == 0) zsh = q;
        else sidx.push_back(q);
    }
    int* d_sidx = nullptr;
    CKS(B.put(&d_sidx, sidx.data(), sidx.size(), st));
    p.sidx = d_sidx;
    p.nsh2 = (int)sidx.size();
    p.zsh = zsh;
    auto blocks = [](long long t) { return (unsigned)((t + ES_NT - 1) / ES_NT); };
    if (ncomp > 0) {
        es_phase_kernel<<<blocks((long long)ns * ncomp), ES_NT, 0, st>>>(p, shf);
        if (in->kernel_kind == 0)
            es_slice_kernel<0><<<blocks((long long)npose * ncomp), ES_NT, 0, st>>>(p);
        else
            es_slice_kernel<1><<<blocks((long long)npose * ncomp), ES_NT, 0, st>>>(p);
    }
    std::vector<int> hcnt;
    std::vector<long long> hoff;
    int* dcand = nullptr;
    double* dw = nullptr;
    size_t dcap = 0;
    for (int b0 = 0; b0 < np; b0 += nb) {
        const int m = std::min(nb, np - b0);
        if (host_images) {
            if (cudaMemcpyAsync(img_b, in->images + (size_t)b0 * n * n * 2, sizeof(double2) * (size_t)m * n * n,
                                cudaMemcpyHostToDevice, st) != cudaSuccess ||
                cudaMemcpyAsync(ip_b, in->image_params + (size_t)b0 * 6, sizeof(double) * (size_t)m * 6,
                                cudaMemcpyHostToDevice, st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "e_step: image upload failed");
            p.img = img_b;
            p.ip = ip_b;
        } else {
            p.img = resident->img + (size_t)b0 * n * n;
            p.ip = resident->ip + (size_t)b0 * 6;
        }
        p.npart = m;
        es_ptab_kernel<<<m, ES_NT, 0, st>>>(p);
        es_pass1_kernel<<<(unsigned)((size_t)m * npose), ES_NT, 0, st>>>(p);
        es_min_kernel<<<m, ES_NT, 0, st>>>(p);
        es_pass2_kernel<<<(unsigned)((size_t)m * ((npose + ES_PG - 1) / ES_PG)), ES_NT, 0, st>>>(p);
        es_softmax_kernel<<<m, ES_NT, 0, st>>>(p, post);
        if (cudaGetLastError() != cudaSuccess) return fail(CM_ERR_CUDA, "e_step: launch failed");
        if (sink.dense) {
            if (cudaMemcpyAsync(sink.dense + (size_t)b0 * nc, post, sizeof(double) * m * nc,
                                cudaMemcpyDeviceToHost, st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "e_step: download failed");
            continue;
        }
        // sparse: per-row counts -> offsets -> ordered compaction
        es_count_kernel<<<m, ES_NT, 0, st>>>(post, (int)nc, cnt);
        hcnt.resize(m);
        hoff.resize(m);
        if (cudaMemcpyAsync(hcnt.data(), cnt, sizeof(int) * m, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return fail(CM_ERR_CUDA, "e_step: kernel failed");
        long long tot = 0;
        for (int q = 0; q < m; ++q) {
            hoff[q] = tot;
            tot += hcnt[q];
            sink.row_ptr[b0 + q + 1] = sink.nnz + tot;
        }
        if (sink.overflow || sink.nnz + tot > sink.cap) {
            sink.overflow = true;
            sink.nnz += tot;
            continue;
        }
        if ((size_t)tot > dcap) {
            dcap = std::max<size_t>((size_t)tot, 2 * dcap);
            CKS(B.put(&dcand, (const int*)nullptr, dcap, st));
            CKS(B.put(&dw, (const double*)nullptr, dcap, st));
        }
        if (tot > 0) {
            if (cudaMemcpyAsync(offd, hoff.data(), sizeof(long long) * m, cudaMemcpyHostToDevice, st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "e_step: upload failed");
            es_compact_kernel<<<m, ES_NT, 0, st>>>(post, (int)nc, offd, dcand, dw);
            if (cudaMemcpyAsync(sink.cand + sink.nnz, dcand, sizeof(int) * tot, cudaMemcpyDeviceToHost, st) !=
                    cudaSuccess ||
                cudaMemcpyAsync(sink.weight + sink.nnz, dw, sizeof(double) * tot, cudaMemcpyDeviceToHost, st) !=
                    cudaSuccess ||
                cudaStreamSynchronize(st) != cudaSuccess)
                return fail(CM_ERR_CUDA, "e_step: download failed");
        }
        sink.nnz += tot;
    }
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(CM_ERR_CUDA, "e_step: kernel failed");
    if (sink.overflow)
        return fail(CM_ERR_INVALID_ARGUMENT, "e_step: entry capacity too small (*nnz holds the entries needed)");
    return CM_OK;
}

} // namespace cm
